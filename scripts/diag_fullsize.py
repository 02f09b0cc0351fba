"""Diagnosis: full-size (c3 or c2) step, engine fp32 and bf16 grads vs the numpy oracle.
python scripts/diag_fullsize.py [c3|c2|c3small] [ragged 0|1] [dropout]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import minmt_oracle as O  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Batch, Model, ModelConfig, Rng  # noqa: E402

CF = {"c3": (50000, 1024, 1024, 4, 128, 50, 50), "c2": (30000, 512, 512, 2, 64, 50, 50),
      "c3small": (50000, 1024, 1024, 4, 16, 50, 50), "h1024b16l1": (5000, 1024, 1024, 1, 16, 20, 20),
      "h512b128": (5000, 512, 512, 2, 128, 20, 20), "h1024b128l1": (5000, 1024, 1024, 1, 128, 20, 20)}
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
ragged = bool(int(sys.argv[2])) if len(sys.argv) > 2 else True
p = float(sys.argv[3]) if len(sys.argv) > 3 else 0.2
V, E, H, L, B, S, T = CF[name]
cfg = ModelConfig(V, E, H, L, p)
model = Model.new(cfg, Rng(1))
params = {b.name: b.var.data.copy() for b in model.params.blocks()}
src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=2, ragged=ragged)
t0 = time.time()
d = O.Dims(V, E, H, L, p)
ol, og, _ = O.forward_backward({k: v.copy() for k, v in params.items()}, d, src, sm, tgt, tm, 0.1,
                               gen=np.random.Generator(np.random.PCG64(5)))
print(f"oracle loss {ol:.6f} ({time.time() - t0:.1f} s)")
for mode in ("fp32", "bf16"):
    eng = Engine(cfg, mode=mode)
    for kv in filter(None, os.environ.get("CMT_OPTIONS", "").split(",")):
        k, v = kv.split("=")
        eng.set_option(k, int(v))
    eng.upload(params)
    loss, _ = eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, np.random.Generator(np.random.PCG64(5)),
                       update=False)
    g = eng.grads()
    eng.close()
    errs = {n: O.norm_rel_err(g[n], og[n]) for n in og}
    worst = sorted(errs.items(), key=lambda x: -x[1])[:6]
    print(f"{mode}: loss {loss:.6f} rel {abs(loss - ol) / ol:.2e}; worst blocks", [(n, f"{e:.2e}") for n, e in worst])
    print("   ", {n: f"{errs[n]:.1e}" for n in ("out.w", "out.b", "att.w_c.w", "att.w_a.w", f"dec.l{L}.w_i",
                                                 "dec.l1.w_i", "enc.l1.fwd.w_i", "src_embed")})
