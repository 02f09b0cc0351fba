"""Host-side cost of one end-to-end step (stage: host validation + segment
sort + H2D enqueue; launch: enqueueing the step; wait: device completion)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Model, ModelConfig, Rng  # noqa: E402

V, E, H, L, B, S, T = bench.CONFIGS["c3"]
cfg = ModelConfig(V, E, H, L, 0.2)
eng = Engine(cfg, mode="bf16")
eng.upload(Model.new(cfg, Rng(1)).params)
src, sm, tgt, tm = bench.synthetic_batch(V, S, T, B, seed=0)
rng = Rng(5)
for _ in range(3):
    eng.stage(src, sm, tgt, tm)
    eng.run(1.0, 5.0, 0.1, rng)
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    eng.stage(src, sm, tgt, tm)
    t1 = time.perf_counter()
    eng.run(1.0, 5.0, 0.1, rng, asynchronous=True)
    t2 = time.perf_counter()
    eng.wait()
    t3 = time.perf_counter()
    ts.append((t1 - t0, t2 - t1, t3 - t2, t3 - t0))
import numpy as np  # noqa: E402
a = np.median(np.array(ts), axis=0) * 1e3
print(f"stage {a[0]:.3f} ms  launch {a[1]:.3f} ms  wait {a[2]:.3f} ms  total {a[3]:.3f} ms")
