#!/bin/bash
# One ncu --set full capture per kernel class of a c3 step (scripts/ncu_step.py),
# plus the launch list of a short bench run.  Outputs under gpurun_out/ncu/.
mkdir -p gpurun_out/ncu
cap() {  # name class skip
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -c 1 -f \
    -o gpurun_out/ncu/$1 python scripts/ncu_step.py $2 $3 > gpurun_out/ncu/$1.log 2>&1
  echo "$1 rc=$?"
}
cap bptt_pair 1 1
cap fwd_pair 2 1
cap logits_gemm 0 0
cap ux_gemm 3 3
cap dx_gemm 4 2
cap dw_gemm 5 2
cap dwo_gemm 11 0
cap ce_stats 6 0
cap ce_grad 7 0
cap dropout_mask 8 2
cap dropout_apply 13 2
cap segments 14 0
cap att_scores 9 0
cap sgd_dense 10 0
cap scatter 12 0
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/ncu/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu/launches_bench.log 2>&1
echo "launches rc=$?"
