"""Per-step phase trace of CTA 0 of one forward scan (debug option trace_layer).
Slots: 0 first h stage issued, 4 last issued, 5 MMA saw first stage, 6 MMA saw
last stage, 1 epilogue saw the accumulator, 2 cell done, 3 h_t published.
python scripts/trace_tm.py [layer] [opt=val ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from bench import synthetic_batch
from paper_1802_07170_b200.engine import Engine
from paper_1802_07170_b200.model import ModelConfig
layer = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = ModelConfig(50000, 1024, 1024, 4, 0.2)
eng = Engine(cfg, mode="bf16")
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    eng.set_option(k, int(v))
gen = np.random.default_rng(0)
eng.upload({n: gen.uniform(-0.1, 0.1, size=s).astype(np.float32) for n, s in eng.blocks})
src, sm, tgt, tm = synthetic_batch(50000, 50, 50, 128, 0)
eng.stage(src, sm, tgt, tm)
eng.run(1.0, 5.0, 0.1, None)
eng.set_option("trace_layer", layer)
eng.run(1.0, 5.0, 0.1, None)
T = np.array([eng.stat(f"trace:{i}")[0] for i in range(400)]).reshape(50, 8).astype(np.float64)
med = lambda a: float(np.median(a[2:45])) / 1e3
print(f"layer {layer}: step period us {med(np.diff(T[:, 3])):.2f}")
print(f"  publish(s-1) -> first stage issued {med(T[1:, 0] - T[:-1, 3]):.2f}")
print(f"  first -> last stage issued        {med(T[:, 4] - T[:, 0]):.2f}")
print(f"  first issued -> MMA first stage    {med(T[:, 5] - T[:, 0]):.2f}")
print(f"  last issued -> MMA last stage      {med(T[:, 6] - T[:, 4]):.2f}")
print(f"  MMA last stage -> epilogue tfull   {med(T[:, 1] - T[:, 6]):.2f}")
print(f"  tfull -> cell done                 {med(T[:, 2] - T[:, 1]):.2f}")
print(f"  cell done -> published            {med(T[:, 3] - T[:, 2]):.2f}")
