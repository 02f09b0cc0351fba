#!/bin/bash
# Kernel tests first (short timeout), then the step tests, bench and a launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider > gpurun_out/ktests.txt 2>&1
echo "ktests rc=$?" >> gpurun_out/ktests.txt
tail -3 gpurun_out/ktests.txt
if grep -q "ktests rc=0" gpurun_out/ktests.txt; then
  timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/tests.txt 2>&1
  echo "tests rc=$?" >> gpurun_out/tests.txt; tail -3 gpurun_out/tests.txt
  timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.txt 2>&1
  echo "bench rc=$?" >> gpurun_out/bench.txt; tail -2 gpurun_out/bench.txt
  if [ -n "$LAUNCHES" ]; then
    timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-350} -c ${COUNT:-230} --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
    python scripts/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt 2>&1
    head -30 gpurun_out/launch_summary.txt
  fi
fi
