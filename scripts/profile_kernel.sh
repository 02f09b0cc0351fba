#!/bin/bash
# ncu --set full of one launch of a kernel (regex $1) in the c3 bench, skipping $2 launches of it.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-lstm_fwd_persistent}; S=${2:-2}; OUT=${3:-prof_$K}
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
  -o gpurun_out/$OUT python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/$OUT.log 2>&1
echo "ncu $K rc=$?"
