"""Per-step phase trace of CTA 0 of one backward (BPTT) scan in a c3 step.
python scripts/trace_bwd.py LAYER [opt=val ...]  (LAYER: 100 + layer index)
Slots: 0 round start (ring free), 5 first dU stage issued, 6 last issued,
7 MMA saw last stage, 1 epilogue saw accumulator, 2 partials exchanged,
3 cell done (dU stored), 4 published."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Model, ModelConfig, Rng  # noqa: E402

layer = int(sys.argv[1]) if len(sys.argv) > 1 else 107
V, E, H, L, B, S, T = bench.CONFIGS["c3"]
cfg = ModelConfig(V, E, H, L, 0.2)
eng = Engine(cfg, mode="bf16")
eng.upload(Model.new(cfg, Rng(1)).params)
for a in sys.argv[2:]:
    k, v = a.split("=")
    eng.set_option(k, int(v))
src, sm, tgt, tm = bench.synthetic_batch(V, S, T, B, seed=0)
eng.stage(src, sm, tgt, tm)
rng = Rng(5)
eng.run(1.0, 5.0, 0.1, rng)
eng.set_option("trace_layer", layer)
eng.run(1.0, 5.0, 0.1, rng)
X = np.array([eng.stat(f"trace:{i}")[0] for i in range(51 * 8)]).reshape(51, 8).astype(np.float64)
R = slice(4, 45)
med = lambda a: float(np.median(a[R])) / 1e3
print(f"layer {layer}: step period us {med(np.diff(X[:, 4], prepend=np.nan)):.2f}")
prev4 = np.concatenate([[np.nan], X[:-1, 4]])
print(f"  published(i-1) -> first stage issued {med(X[:, 5] - prev4):.2f}")
print(f"  first -> last stage issued           {med(X[:, 6] - X[:, 5]):.2f}")
print(f"  last issued -> MMA saw last stage    {med(X[:, 7] - X[:, 6]):.2f}")
print(f"  MMA last stage -> epilogue tfull     {med(X[:, 1] - X[:, 7]):.2f}")
print(f"  tfull -> partials exchanged          {med(X[:, 2] - X[:, 1]):.2f}")
print(f"  exchanged -> cell done               {med(X[:, 3] - X[:, 2]):.2f}")
print(f"  cell done -> published               {med(X[:, 4] - X[:, 3]):.2f}")
print(f"  (round start -> first issue          {med(X[:, 5] - X[:, 0]):.2f})")
