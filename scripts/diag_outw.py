"""Diagnosis of the output-layer gradients in bf16 mode at c3-like sizes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import minmt_oracle as O  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Batch, Model, ModelConfig, Rng  # noqa: E402

V, E, H, L, B, S, T = (int(x) for x in (sys.argv[1:8] if len(sys.argv) > 7 else (50000, 1024, 1024, 4, 16, 50, 50)))
p = 0.2
cfg = ModelConfig(V, E, H, L, p)
model = Model.new(cfg, Rng(1))
src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=2, ragged=True)
batch = Batch(src, tgt, sm, tm)
NT = T * B


def run(stop):
    eng = Engine(cfg, mode="bf16")
    eng.upload(model.params)
    if stop:
        eng.set_option("stop_after", stop)
    eng.step(batch, 1.0, 5.0, 0.1, np.random.Generator(np.random.PCG64(5)), update=False)
    Y = eng.debug_buffer("Y", cap=NT * V).reshape(NT, V)
    hod = eng.debug_buffer("hod", cap=NT * H).reshape(NT, H)
    g = eng.grads() if not stop else None
    eng.close()
    return Y, hod, g


logits, hod1, _ = run(1)
dY, hod, g = run(0)
print("hod identical across runs:", np.array_equal(hod1, hod))
y = torch.tensor(logits, dtype=torch.float64)
eps = 0.1
m = torch.tensor(tm.reshape(-1), dtype=torch.float64)
ntok = float(tm.sum())
lp = torch.log_softmax(y, dim=1)
tgt_flat = torch.tensor(tgt.reshape(-1))
d = torch.exp(lp) - eps / V
d[torch.arange(NT), tgt_flat] -= (1 - eps)
d = d * (m / ntok)[:, None] * (1 - y * y)
dYt = torch.tensor(dY, dtype=torch.float64)
print("dY vs float64 recomputation from the engine's logits: norm-rel", O.norm_rel_err(dY, d.numpy()))
ref_w = torch.tensor(hod, dtype=torch.float64).t() @ dYt
print("out.w grad vs hod^T dY(engine):", O.norm_rel_err(g["out.w"], ref_w.numpy()))
ref_w2 = torch.tensor(hod, dtype=torch.float64).t() @ d
print("out.w grad vs hod^T dY(float64):", O.norm_rel_err(g["out.w"], ref_w2.numpy()))
print("hod^T dY(engine) vs hod^T dY(float64):", O.norm_rel_err(ref_w.numpy(), ref_w2.numpy()))
print("out.b grad vs column sums of dY(float64):", O.norm_rel_err(g["out.b"].ravel(), d.sum(0).numpy()))
print("max|dY| non-gold ~", float(d.abs().median()), " gold ~", float(d[torch.arange(NT), tgt_flat].abs().mean()))
