"""Run c3 train steps with one kernel class marked for ncu.

    ncu --profile-from-start off --set full --clock-control none --import-source on \
        -c 1 -o gpurun_out/<name> python scripts/ncu_step.py CLASS [SKIP] [config]

The engine wraps the first launch of CLASS in the profiled step with
cudaProfilerStart/Stop (engine option ncu_class), so `-c 1` captures exactly
that kernel: 0 logits GEMM, 1 BPTT scan, 2 forward scan, 3 Ux GEMM, 4 dX GEMM,
5 dW GEMM, 6 ce_stats, 7 ce_grad, 8 dropout, 9 attention scores GEMM,
10 dense SGD, 11 dW_o GEMM, 12 embedding scatter, 13 dropout apply, 14 embedding
segments (8 is the dropout mask kernel when masks are generated ahead).  One warm step runs first
(unmarked), so the capture sees a hot engine.  Under ncu the recurrent scans
launch non-cooperatively (the engine detects the profiler).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Model, ModelConfig, Rng  # noqa: E402

cls = int(sys.argv[1])
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # launches of the class to pass over
name = sys.argv[3] if len(sys.argv) > 3 else "c3"
V, E, H, L, B, S, T = bench.CONFIGS[name]
cfg = ModelConfig(V, E, H, L, 0.2)
eng = Engine(cfg, mode="bf16")
eng.upload(Model.new(cfg, Rng(1)).params)
src, sm, tgt, tm = bench.synthetic_batch(V, S, T, B, seed=0)
eng.stage(src, sm, tgt, tm)
rng = Rng(5)
eng.run(1.0, 5.0, 0.1, rng)
eng.set_option("ncu_skip", skip)
eng.set_option("ncu_class", cls)
eng.run(1.0, 5.0, 0.1, rng)
print("done")
