"""Per-launch device timeline of one beam-10 decode step at c3 (debug)."""
import os, sys, time, collections
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1802_07170_b200.engine import Engine
from paper_1802_07170_b200.model import Model, ModelConfig, Rng
cfg = ModelConfig(50000, 1024, 1024, 4, 0.2)
model = Model.new(cfg, Rng(1))
eng = Engine(cfg, mode="bf16"); eng.upload(model.params)
src = list(range(4, 54))
eng.decode_begin(src)
v, t = eng.decode_step([2], None, 10)
prev = [int(x) for x in t[0]]
for _ in range(3): v, t = eng.decode_step(prev, list(range(10)) if _ else [0]*10, 10)
eng.set_option("timeline", 1)
t0 = time.perf_counter()
for _ in range(20): eng.decode_step(prev, list(range(10)), 10)
dt = (time.perf_counter() - t0) / 20
tl = eng.timeline(); eng.set_option("timeline", 0)
agg = collections.defaultdict(float)
for lab, ms in tl: agg[lab] += ms / 20
print(f"wall per step {dt*1e3:.3f} ms; device sum {sum(agg.values()):.3f} ms")
for k, v in sorted(agg.items(), key=lambda x: -x[1]): print(f"  {v*1e3:8.1f} us {k}")
