"""bf16 vs fp32 engine forward activations (stop after the logits GEMM)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import minmt_oracle as O  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Batch, Model, ModelConfig, Rng  # noqa: E402

V, E, H, L, B, S, T = (int(x) for x in (sys.argv[1:8] if len(sys.argv) > 7 else (50000, 1024, 1024, 4, 16, 50, 50)))
p = float(sys.argv[8]) if len(sys.argv) > 8 else 0.2
cfg = ModelConfig(V, E, H, L, p)
model = Model.new(cfg, Rng(1))
src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=2, ragged=True)
batch = Batch(src, tgt, sm, tm)
NT, NS = T * B, S * B
names = ["Xs", "Xt"] + [f"yext:{l}" for l in range(2 * L + 1)] + ["u_att", "alpha", "cst_att", "ho", "Y"]
out = {}
for mode in ("fp32", "bf16"):
    eng = Engine(cfg, mode=mode)
    eng.upload(model.params)
    eng.set_option("stop_after", 1)
    eng.step(batch, 1.0, 5.0, 0.1, np.random.Generator(np.random.PCG64(5)), update=False)
    out[mode] = {n: eng.debug_buffer(n, cap=NT * V + 16) for n in names}
    eng.close()
for n in names:
    a, b = out["fp32"][n], out["bf16"][n]
    print(f"{n:10s} norm-rel {O.norm_rel_err(b, a):.3e}   rms-rel {np.sqrt(np.mean((a - b) ** 2) / max(np.mean(a * a), 1e-30)):.3e}  |a|max {np.abs(a).max():.3e}")
