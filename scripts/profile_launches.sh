#!/bin/bash
# Launch list (cold-cache, serialised) of one c3 bench step: gpu__time_duration per kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SKIP=${SKIP:-3200}
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $SKIP -c ${COUNT:-1100} --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo "ncu rc=$?"
