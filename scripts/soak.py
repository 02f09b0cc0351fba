"""Soak run: N c3 train steps through the reference-signature train_step with a
new synthetic batch every step (ragged masks, fresh ids, so every replay of the
captured step graph sees different ids, masks and unique-row counts), random-init
weights, dropout 0.2, clip 5.  Reports the loss trend, wall time and
how many steps replayed the graph; fails on any error or non-finite loss.

The batches repeat a small pool of source/target sequences so the model can
fit them and the loss visibly falls (a learning check, not only a stability one).

python scripts/soak.py [steps] [config]
"""
import json
import os
import sys
import time
import types

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1802_07170_b200 import training as TR  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Batch, Model, ModelConfig, Rng  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 400
name = sys.argv[2] if len(sys.argv) > 2 else "c3"
V, E, H, L, B, S, T = bench.CONFIGS[name]
cfg = ModelConfig(V, E, H, L, 0.2)
model = Model.new(cfg, Rng(1))
eng = Engine(cfg, mode="bf16")
eng.upload(model.params)
TR._ENGINES[model] = eng
tcfg = types.SimpleNamespace(grad_clip_norm=5.0, label_smoothing=0.1)
rng = Rng(7)
g = np.random.default_rng(0)
pool = 8 * B  # sentence pool
src_pool = g.integers(4, V, size=(S, pool))
tgt_pool = g.integers(4, V, size=(T, pool))
losses = []
t0 = time.perf_counter()
for i in range(steps):
    cols = g.choice(pool, size=B, replace=False)
    src, tgt = src_pool[:, cols].copy(), tgt_pool[:, cols].copy()
    ls = g.integers(S // 2, S + 1, size=B)
    lt = g.integers(T // 2, T + 1, size=B)
    sm = (np.arange(S)[:, None] < ls[None, :]).astype(np.float32)
    tm = (np.arange(T)[:, None] < lt[None, :]).astype(np.float32)
    loss = TR.train_step(model, Batch(src, tgt, sm, tm), tcfg, 0.5, rng, sync="lazy")
    if not np.isfinite(loss):
        raise SystemExit(f"non-finite loss at step {i}")
    losses.append(float(loss))
dt = time.perf_counter() - t0
replays = eng.stat("graph_replays")[0]
k = max(1, steps // 10)
print(json.dumps({"config": name, "steps": steps, "seconds": round(dt, 2), "ms_per_step_wall": round(1e3 * dt / steps, 3),
                  "graph_replays": int(replays), "loss_first10": round(float(np.mean(losses[:k])), 4),
                  "loss_last10": round(float(np.mean(losses[-k:])), 4),
                  "loss_every_10pct": [round(float(np.mean(losses[j:j + k])), 3) for j in range(0, steps, k)]}))
