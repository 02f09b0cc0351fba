import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import minmt_oracle as O  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from tests.gpu_helpers import cfg_of, scaled_params  # noqa: E402

V, E, H, L, B, S, T = (1000, 128, 128, 1, 16, 9, 8)
d = O.Dims(V, E, H, L, 0.0)
params = scaled_params(d, 3, 0.1)
src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=4, ragged=True)
loss, _, aux = O.forward_backward({k: v.copy() for k, v in params.items()}, d, src, sm, tgt, tm, 0.1,
                                  want_grads=False)
ref_logits = aux["logits"].T.ravel()  # token-major
for stop in [1, 2]:
    outs = []
    for mode in ["fp32", "bf16", "bf16", "bf16"]:
        eng = Engine(cfg_of(d), mode=mode)
        eng.upload(params)
        eng.set_option("stop_after", stop)
        eng.stage(src, sm, tgt, tm)
        try:
            eng.run(1.0, 5.0, 0.1, None, update=False)
        except Exception as ex:
            print("run exc", ex)
        outs.append(eng.debug_buffer("Y"))
        eng.close()
    print("stop", stop, "fp32 vs oracle logits", O.norm_rel_err(outs[0], ref_logits) if stop == 1 else "-",
          "bf16 vs fp32", [f"{O.norm_rel_err(o, outs[0]):.2e}" for o in outs[1:]], flush=True)
    if stop == 1:
        b = outs[1].reshape(B * T, V)
        f = outs[0].reshape(B * T, V)
        bad = np.argwhere(np.abs(b - f) > 0.05 * np.abs(f).max())
        print("bad count", len(bad), bad[:20].tolist())
