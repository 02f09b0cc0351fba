#!/bin/bash
# Step-level GPU checks: persistent/dual parity test, all gpu tests, timeline, bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_step.py -q -x -p no:cacheprovider -k "persistent_recurrence" > gpurun_out/ptests.txt 2>&1
echo "ptests rc=$?" >> gpurun_out/ptests.txt; tail -3 gpurun_out/ptests.txt
if grep -q "ptests rc=0" gpurun_out/ptests.txt; then
  timeout -s KILL 200 python scripts/timeline.py c3 $TLOPTS > gpurun_out/timeline_c3.txt 2>&1; head -24 gpurun_out/timeline_c3.txt
  timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.txt 2>&1; tail -1 gpurun_out/bench.txt | cut -c1-400
  if [ -n "$ALL" ]; then
    timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/tests.txt 2>&1
    echo "tests rc=$?" >> gpurun_out/tests.txt; tail -3 gpurun_out/tests.txt
  fi
fi
