"""Full-size checks at BASELINE.json's single-GPU configurations (configs[2]
c3: 4x1024, V=50k, B=128, S=T=50; configs[4] c5: 2x1024, V=100k, B=256,
S=T=80), where the numpy oracle would take minutes per step: size-independent
properties instead.

* bf16 production mode vs the engine's fp32 validation mode (SIMT GEMMs, the
  mode pinned to the reference's own outputs by test_gpu_step.py): loss and
  every block's gradient within the 2e-2 norm-relative tolerance, with the
  weights at 1/4 of the reference init.  At the reference init itself the
  1024-wide 4-layer recurrence is expanding: rounding only the WEIGHTS to bf16
  (fp32 engine) moves H_o by 17 % rms and a 1e-4 input perturbation grows 15x
  (scripts/diag_chaos.py, profiles/r01/s3/fullsize_sensitivity.txt), so no
  bf16 implementation can meet 2e-2 there; at 1/4 scale the same rounding
  moves H_o by 0.4 %.
* At initialisation the tanh-bounded logits make the prediction nearly
  uniform: the smoothed loss is close to log V (the reference's known answer
  for uniform predictions, pkg/tests/test_training.py:36-41).
* Bitwise determinism of the bf16 step (losses, grads, rng state).
* The update: w_new = w - fp32(lr * scale) * g with the reported norm.
"""

import math

import numpy as np
import pytest

from oracle import minmt_oracle as O

pytestmark = pytest.mark.gpu

CONFIGS = {"c3": (50000, 1024, 1024, 4, 128, 50, 50), "c5": (100000, 1024, 1024, 2, 256, 80, 80)}
TOL = 2e-2


@pytest.mark.parametrize("name", list(CONFIGS))
def test_fullsize_bf16_vs_fp32_and_properties(name):
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch, Model, ModelConfig, Rng
    V, E, H, L, B, S, T = CONFIGS[name]
    cfg = ModelConfig(V, E, H, L, 0.2)
    model = Model.new(cfg, Rng(1))
    src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=2, ragged=True)
    batch = Batch(src, tgt, sm, tm)
    quarter = {b.name: (0.25 * b.var.data).astype(np.float32) for b in model.params.blocks()}
    res = {}
    for mode in ("fp32", "bf16", "bf16"):
        eng = Engine(cfg, mode=mode)
        eng.upload(quarter)
        gen = np.random.Generator(np.random.PCG64(5))
        loss, _ = eng.step(batch, 1.0, 5.0, 0.1, gen, update=False)
        res.setdefault(mode, []).append((loss, eng.grads(), gen.bit_generator.state))
        eng.close()
    (lf, gf, sf), = res["fp32"]
    (lb, gb, sb), (lb2, gb2, sb2) = res["bf16"]
    assert abs(lb - lf) <= TOL * abs(lf)
    errs = {n: O.norm_rel_err(gb[n], gf[n]) for n in gf}
    assert max(errs.values()) < TOL, {n: e for n, e in errs.items() if e >= TOL}
    assert sf == sb == sb2
    assert lb == lb2
    for n in gb:
        assert np.array_equal(gb[n], gb2[n]), n
    # the reference init: near-uniform prediction (loss ~ log V) and one real
    # update w_new = w - fp32(lr * scale) * g (training.py:123-142)
    eng = Engine(cfg, mode="bf16")
    eng.upload(model.params)
    w0 = {b.name: b.var.data.copy() for b in model.params.blocks()}
    loss0, _ = eng.step(batch, 1.0, 5.0, 0.1, np.random.Generator(np.random.PCG64(5)), update=False)
    gb = eng.grads()
    assert abs(loss0 - math.log(V)) < 0.02 * math.log(V), (loss0, math.log(V))
    lr, clip = 0.5, 0.05  # a small clip so the scale is exercised
    _, norm = eng.step(batch, lr, clip, 0.1, np.random.Generator(np.random.PCG64(5)))
    w1 = eng.params()
    eng.close()
    gnorm = math.sqrt(sum(float(np.dot(g.ravel().astype(np.float64), g.ravel().astype(np.float64)))
                          for g in gb.values()))
    assert abs(norm - gnorm) <= 1e-3 * gnorm
    s32 = np.float32(lr * min(1.0, clip / norm))
    for n in ("out.w", "att.w_c.w", f"dec.l{L}.w_i", "src_embed"):
        exp = w0[n] - s32 * gb[n]
        assert O.norm_rel_err(w1[n] - w0[n], exp - w0[n]) < 1e-5, n
