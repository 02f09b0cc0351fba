"""Localise a bf16-vs-fp32 divergence: run both engines on one batch and compare
every internal buffer in forward/backward order."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import minmt_oracle as O  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Batch  # noqa: E402
from tests.gpu_helpers import cfg_of, scaled_params  # noqa: E402

case = tuple(int(x) for x in sys.argv[1].split(",")) if len(sys.argv) > 1 else (1000, 128, 128, 1, 16, 9, 8)
V, E, H, L, B, S, T = case
d = O.Dims(V, E, H, L, 0.0)
params = scaled_params(d, 3, 0.1)
src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=4, ragged=True)
names = ["Xs", "Xt"] + [f"yext:{l}" for l in range(2 * L + 1)] + [f"cext:{l}" for l in range(2 * L + 1)] + \
        ["top", "u_att", "alpha", "cst_att", "ho", "hod", "Y", "dhpre", "dcst", "du_att"] + \
        [f"dy:{l}" for l in range(2 * L + 1)] + ["dtop", "dXemb"]
bufs = {}
for mode in ["fp32", "bf16", "bf16"]:
    eng = Engine(cfg_of(d), mode=mode)
    eng.upload(params)
    eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, np.random.default_rng(0), update=False)
    got = {n: eng.debug_buffer(n) for n in names}
    key = mode if mode not in bufs else mode + "_2"
    bufs[key] = got
    eng.close()
for n in names:
    a, b, c = bufs["fp32"][n], bufs["bf16"][n], bufs["bf16_2"][n]
    print(f"{n:10s} fp32-vs-bf16 {O.norm_rel_err(b, a):.2e}  bf16 repeat {O.norm_rel_err(c, b):.2e} "
          f" nan={np.isnan(b).sum()} max|fp32|={np.abs(a).max():.3e}", flush=True)
