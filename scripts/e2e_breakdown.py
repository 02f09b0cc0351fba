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

# the reference-signature call, and the device time of the same steps
import types  # noqa: E402
from paper_1802_07170_b200 import training as TR  # noqa: E402
from paper_1802_07170_b200.model import Batch  # noqa: E402
model = Model.new(cfg, Rng(1))
TR._ENGINES[model] = eng
batch = Batch(src, tgt, sm, tm)
tcfg = types.SimpleNamespace(grad_clip_norm=5.0, label_smoothing=0.1)
for _ in range(3):
    TR.train_step(model, batch, tcfg, 1.0, rng, sync="lazy")
for i in range(8):
    eng.stat(f"stage_us:{i}")  # reset the staging phase counters (first-call allocations)
eng.record(0)
t0 = time.perf_counter()
for _ in range(20):
    TR.train_step(model, batch, tcfg, 1.0, rng, sync="lazy")
t1 = time.perf_counter()
eng.record(1)
dev = eng.elapsed_ms(0, 1) / 20
print(f"train_step {1e3 * (t1 - t0) / 20:.3f} ms per call; device span {dev:.3f} ms per call")
import cProfile, pstats  # noqa: E402,E401
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    TR.train_step(model, batch, tcfg, 1.0, rng, sync="lazy")
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
n = eng.stat("stage_us:6")[1]
names = ["validate+ntok", "ensure_ws/layout", "convert+5 H2D", "build keys", "segment sort+3 H2D", "event"]
print("stage phases (us per call):", {nm: round(eng.stat(f"stage_us:{i}")[0] / n, 1) for i, nm in enumerate(names)})
