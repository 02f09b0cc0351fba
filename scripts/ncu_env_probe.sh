#!/bin/bash
# Debug: what does a process see under ncu, and does the BPTT cluster kernel run
# non-cooperatively (CMT_COOP=0) with and without the profiler.
python -c "import os; print({k: v for k, v in os.environ.items() if 'INJECT' in k or 'NSIGHT' in k or 'NV_' in k or 'PRELOAD' in k})" > gpurun_out/env_plain.txt
ncu --metrics gpu__time_duration.sum -c 1 python -c "import os; print({k: v for k, v in os.environ.items() if 'INJECT' in k or 'NSIGHT' in k or 'NV_' in k or 'PRELOAD' in k}); import torch; torch.zeros(1).cuda()" > gpurun_out/env_ncu.txt 2>&1
CMT_COOP=0 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_nocoop.txt 2>&1
CMT_COOP=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_smoke_nocoop.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu_nocoop.txt 2>&1
echo "ncu nocoop rc=$?" >> gpurun_out/smoke_ncu_nocoop.txt
