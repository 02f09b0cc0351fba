"""Parity sweep at full model width.

For a BASELINE config's width (c3: V=50k, E=H=1024, L=4, B=128; c5: V=100k,
L=2, B=256) and a list of sequence lengths S=T, runs one step from the
reference init (Model.new(ModelConfig(...), Rng(1))) with:
  * the numpy oracle in fp32 (the reference algorithm) and in fp64 (its twin,
    reference model.py:129-134) -> the reference's own fp32 floor;
  * the engine in fp32 validation mode and in bf16 production mode.
and prints, per length, loss rel error and the worst per-block norm-relative
gradient error (pkg/tests/helpers.py:80-81) of each against the fp32 oracle
(and of the fp32 oracle against fp64).

python scripts/parity_sweep.py c3 4,8,16,50 [dropout]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import minmt_oracle as O  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Batch, Model, ModelConfig, Rng  # noqa: E402

CF = {"c3": (50000, 1024, 1024, 4, 128), "c5": (100000, 1024, 1024, 2, 256), "c2": (30000, 512, 512, 2, 64)}


def worst(errs, k=4):
    return [(n, float(f"{e:.2e}")) for n, e in sorted(errs.items(), key=lambda x: -x[1])[:k]]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    lens = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "8").split(",")]
    p = float(sys.argv[3]) if len(sys.argv) > 3 else 0.2
    modes = os.environ.get("SWEEP_MODES", "fp64,bf16w,fp32,bf16").split(",")
    V, E, H, L, B = CF[name]
    cfg = ModelConfig(V, E, H, L, p)
    d = O.Dims(V, E, H, L, p)
    model = Model.new(cfg, Rng(1))
    params = {b.name: b.var.data.copy() for b in model.params.blocks()}
    out = []
    for n in lens:
        src, sm, tgt, tm = O.synthetic_batch(V, n, n, B, seed=2, ragged=True)
        t0 = time.time()
        ol, og, _ = O.forward_backward({k: v.copy() for k, v in params.items()}, d, src, sm, tgt, tm, 0.1,
                                       gen=np.random.Generator(np.random.PCG64(5)))
        row = {"config": name, "S=T": n, "B": B, "oracle_fp32_s": round(time.time() - t0, 1), "loss": ol}
        g64 = None
        if "fp64" in modes:
            t0 = time.time()
            l64, g64, _ = O.forward_backward({k: v.astype(np.float64) for k, v in params.items()}, d, src, sm, tgt,
                                             tm, 0.1, gen=np.random.Generator(np.random.PCG64(5)))
            e = {k: O.norm_rel_err(og[k], g64[k]) for k in og}
            row["oracle_fp32_vs_fp64"] = {"loss_rel": abs(ol - l64) / abs(l64), "worst": worst(e),
                                          "max": max(e.values())}
        if "bf16w" in modes:
            # the reference algorithm in fp32 on the bf16-rounded weights: how far
            # merely storing the weights in bf16 moves the reference's own step
            import torch
            pw = {k: torch.from_numpy(v).to(torch.bfloat16).float().numpy() for k, v in params.items()}
            lw_, gw, _ = O.forward_backward(pw, d, src, sm, tgt, tm, 0.1, gen=np.random.Generator(np.random.PCG64(5)))
            e = {k: O.norm_rel_err(gw[k], og[k]) for k in og}
            row["oracle_bf16_weights_vs_oracle"] = {"loss_rel": abs(lw_ - ol) / abs(ol), "worst": worst(e),
                                                    "max": max(e.values())}
            del gw
        for mode in ("fp32", "bf16"):
            if mode not in modes:
                continue
            eng = Engine(cfg, mode=mode)
            eng.upload(params)
            loss, _ = eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, np.random.Generator(np.random.PCG64(5)),
                               update=False)
            g = eng.grads()
            eng.close()
            e = {k: O.norm_rel_err(g[k], og[k]) for k in og}
            row[f"engine_{mode}_vs_oracle"] = {"loss_rel": abs(loss - ol) / abs(ol), "worst": worst(e),
                                               "max": max(e.values())}
            if g64 is not None:
                e = {k: O.norm_rel_err(g[k], g64[k]) for k in og}
                row[f"engine_{mode}_vs_fp64"] = {"worst": worst(e, 2), "max": max(e.values())}
        print(json.dumps(row), flush=True)
        out.append(row)
    return out


if __name__ == "__main__":
    main()
