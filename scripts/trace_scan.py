"""Per-step phase timestamps (globaltimer) of CTA 0 of one recurrent scan in a
c3 step.  python scripts/trace_scan.py LAYER   (LAYER >= 100: backward scan of layer LAYER-100)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Model, ModelConfig, Rng  # noqa: E402

layer = int(sys.argv[1]) if len(sys.argv) > 1 else 102
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
names = ["t0", "t1", "t2", "t3", "t4", "t5", "t6", "t7"]
rows = slice(3, 40)
if layer < 100:
    # fwd multi: 4 first stage issued, 5 last stage issued, 6 first stage landed (MMA),
    # 7 last stage landed, 1 tfull (epilogue), 2 cell done, 3 published
    seq = [(3, "published(prev)"), (4, "first issue"), (5, "last issue"), (6, "first landed"), (7, "last landed"),
           (1, "tfull"), (2, "cell done"), (3, "published")]
    R = X[1:][rows]
    P = X[:-1][rows]
    prev = P[:, 3]
    for col, nm in seq[1:]:
        cur = R[:, col]
        print(f"  {nm:14s} +{np.median(cur - prev) / 1e3:6.2f} us")
        prev = cur
per = np.diff(X[:, 0])[rows]
print(f"layer {layer}: step period us median {np.median(per) / 1e3:.2f}")
for a, b in [(0, 1), (1, 2), (2, 3), (3, 4)]:
    d = (X[:, b] - X[:, a])[rows] / 1e3
    if np.all(X[rows, a] > 0) and np.all(X[rows, b] > 0):
        print(f"  {names[a]}->{names[b]} us median {np.median(d):.2f}")
d = (X[1:, 0] - X[:-1, 4])[rows] / 1e3
print(f"  t4->next t0 us median {np.median(d):.2f}")
d = (X[1:, 0] - X[:-1, 3])[rows] / 1e3
print(f"  t3->next t0 us median {np.median(d):.2f}")

if layer >= 100:
    Y = np.array([eng.stat(f"trace:{1024 + i}")[0] for i in range(51 * 8)]).reshape(51, 8).astype(np.float64)
    if Y[5, 0] > 0:
        rel = (Y - Y[:, :1])[rows] / 1e3
        print("  tfull of CTAs 0..7 relative to CTA 0 (us), median:", np.round(np.median(rel, axis=0), 2))
        print("  max spread within cluster 0 (us), median:", np.median(rel[:, :4].max(1) - rel[:, :4].min(1)))
