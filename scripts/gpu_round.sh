#!/bin/bash
# Round evidence on one GPU box: gpu tests, smoke, default bench, timeline,
# ncu launch list of one bench step, ncu --set full of the named kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests.txt; tail -3 gpurun_out/tests.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout -s KILL 600 python bench.py > gpurun_out/bench.txt 2>&1; tail -1 gpurun_out/bench.txt | cut -c1-200
timeout -s KILL 200 python scripts/timeline.py c3 > gpurun_out/timeline_c3.txt 2>&1; head -3 gpurun_out/timeline_c3.txt
if [ -n "$LAUNCHES" ]; then
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-400} -c ${COUNT:-130} --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
  echo "ncu launches rc=$?"; tail -3 gpurun_out/ncu_launches.log
fi
for K in $FULL; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$K -s ${FSKIP:-3} -c 1 \
    -o gpurun_out/full_$K python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$K.log 2>&1
  echo "ncu full $K rc=$?"; tail -2 gpurun_out/ncu_full_$K.log
done
