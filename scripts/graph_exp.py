"""EXPERIMENT: device time per c3 step, eager launches vs one captured CUDA graph replayed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1802_07170_b200.engine import Engine
from paper_1802_07170_b200.model import Model, ModelConfig, Rng
import bench

cfg = ModelConfig(50000, 1024, 1024, 4, 0.2)
model = Model.new(cfg, Rng(1))
eng = Engine(cfg, mode="bf16")
eng.upload(model.params)
src, sm, tgt, tm = bench.synthetic_batch(50000, 50, 50, 128, seed=0)
eng.stage(src, sm, tgt, tm)
rng = Rng(5)
for mode in (0, 1, 0, 1):
    eng.set_option("graph_exp", mode)
    for _ in range(3):
        eng.run(1.0, 5.0, 0.1, rng)
    eng.record(0)
    for _ in range(30):
        eng.run(1.0, 5.0, 0.1, rng, asynchronous=True)
    eng.record(1)
    eng.wait()
    print("graph" if mode else "eager", round(eng.elapsed_ms(0, 1) / 30, 4), "ms/step", flush=True)
