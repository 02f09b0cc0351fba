#!/bin/bash
# One GPU-box session: tests, smoke, bench.  Each stage is wrapped in its own timeout.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
timeout -s KILL ${T_TESTS:-900} python -m pytest tests -m "${PYTEST_MARK:-gpu}" -q --maxfail=15 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.txt
if [ -n "$BENCH" ]; then
  timeout -s KILL ${T_BENCH:-600} python bench.py $BENCH > gpurun_out/bench.txt 2>&1
  echo "bench rc=$?" >> gpurun_out/bench.txt
fi
tail -5 gpurun_out/tests.txt; tail -3 gpurun_out/smoke.txt; tail -3 gpurun_out/bench.txt 2>/dev/null
