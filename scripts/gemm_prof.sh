#!/bin/bash
# GEMM micro-benchmark + one ncu --set full capture of the logits GEMM (tile $1, default 257).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 300 python scripts/gemm_bench.py > gpurun_out/gemm_bench.txt 2>&1; echo "gemm_bench rc=$?" >> gpurun_out/gemm_bench.txt
cat gpurun_out/gemm_bench.txt
if [ -n "$PROF" ]; then
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 \
  -o gpurun_out/prof_gemm_logits python scripts/gemm_bench.py --only logits --tiles ${1:-257} --iters 1 > gpurun_out/prof_gemm.log 2>&1
echo "ncu rc=$?"
fi
