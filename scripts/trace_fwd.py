import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from bench import synthetic_batch
from paper_1802_07170_b200.engine import Engine
from paper_1802_07170_b200.model import Model, ModelConfig, Rng
cfg = ModelConfig(50000, 1024, 1024, 4, 0.2)
eng = Engine(cfg, mode="bf16")
gen = np.random.default_rng(0)
eng.upload({n: gen.uniform(-0.1, 0.1, size=s).astype(np.float32) for n, s in eng.blocks})
src, sm, tgt, tm = synthetic_batch(50000, 50, 50, 128, 0)
eng.stage(src, sm, tgt, tm)
eng.run(1.0, 5.0, 0.1, None)
eng.set_option("trace_layer", 2)
eng.run(1.0, 5.0, 0.1, None)
T = np.array([eng.stat(f"trace:{i}")[0] for i in range(400)]).reshape(50, 8)
d = np.diff(T.reshape(-1))
T0 = T[:, 0]
print("step period us", np.diff(T0)[1:10] / 1e3)
print("acquire->tfull us", (T[:, 1] - T[:, 0])[1:10] / 1e3)
print("tfull->epi done us", (T[:, 2] - T[:, 1])[1:10] / 1e3)
print("epi done->signal us", (T[:, 3] - T[:, 2])[1:10] / 1e3)
print("signal->next acquire us", (T[1:, 0] - T[:-1, 3])[1:10] / 1e3)
print("acquire->full0 us", (T[:, 4] - T[:, 0])[1:10] / 1e3)
print("full0->full5 us", (T[:, 5] - T[:, 4])[1:10] / 1e3)
print("full5->full6 us", (T[:, 6] - T[:, 5])[1:10] / 1e3)
print("full6->full15 us", (T[:, 7] - T[:, 6])[1:10] / 1e3)
print("full15->tfull us", (T[:, 1] - T[:, 7])[1:10] / 1e3)
