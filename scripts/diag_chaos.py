"""Sensitivity of the c3-size forward to a tiny perturbation (fp32 engine vs fp32 engine with the
source embeddings perturbed by 1e-4 relative, and by bf16 rounding of all weights), at the reference
init scale and at 1/4 of it: a chaotic (expanding) recurrence amplifies the perturbation."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import minmt_oracle as O  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Batch, Model, ModelConfig, Rng  # noqa: E402

V, E, H, L, B, S, T = 50000, 1024, 1024, 4, 16, 50, 50
cfg = ModelConfig(V, E, H, L, 0.2)
src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=2, ragged=True)
batch = Batch(src, tgt, sm, tm)
names = ["yext:0", "yext:4", "yext:8", "ho"]
g = np.random.default_rng(7)
for scale in (1.0, 0.25):
    model = Model.new(cfg, Rng(1))
    base = {b.name: (b.var.data * scale).astype(np.float32) for b in model.params.blocks()}
    runs = {}
    for tag in ("ref", "perturbed", "bf16-rounded"):
        p = {k: v.copy() for k, v in base.items()}
        if tag == "perturbed":
            p["src_embed"] *= (1 + 1e-4 * g.standard_normal(p["src_embed"].shape)).astype(np.float32)
        if tag == "bf16-rounded":
            import torch
            p = {k: torch.tensor(v).bfloat16().float().numpy() for k, v in p.items()}
        eng = Engine(cfg, mode="fp32")
        eng.upload(p)
        eng.set_option("stop_after", 1)
        eng.step(batch, 1.0, 5.0, 0.1, np.random.Generator(np.random.PCG64(5)), update=False)
        runs[tag] = {n: eng.debug_buffer(n, cap=(T + 1) * B * H + 16) for n in names}
        eng.close()
    for tag in ("perturbed", "bf16-rounded"):
        print(f"init x{scale} {tag:13s}", "  ".join(
            f"{n} rms-rel {np.sqrt(np.mean((runs[tag][n] - runs['ref'][n]) ** 2) / np.mean(runs['ref'][n] ** 2)):.2e}"
            for n in names))
