"""Parity at the widths bench.py reports (BASELINE.json configs[2] c3:
4x1024, V=50k, B=128 and configs[4] c5: 2x1024, V=100k, B=256), from the
reference init ``Model.new(ModelConfig(...), Rng(1))`` (uniform +-0.1, forget
bias 1), against the numpy oracle (the reference algorithm, pinned to the
reference's own outputs by tests/test_oracle.py).

* Full width, short sequences (S=T=8): the north-star tolerances hold as
  stated — fp32 validation mode 1e-4 and bf16 production mode 2e-2,
  norm-relative (pkg/tests/helpers.py:80-81) — on the loss, every block's
  gradient, the gradient norm and the updated weights; the dropout generator
  ends in the reference's state.  These sizes run the V=50k/100k CE, the
  256-wide CTA-pair GEMM tiles, the 128-row recurrent slices and every
  production kernel of the bench step.
* Full length (c3, S=T=50): the reference itself is sensitive there.  Its own
  fp32 step differs from its exact fp64 twin (reference model.py:129-134) by
  ~2e-4 (worst block) and merely rounding the initial weights to bf16 moves
  its gradients by O(1) (scripts/parity_sweep.py,
  profiles/r02/parity_sweep.txt).  The stated tolerance is below the
  reference's own floor at that length, so the test states the attainable
  one: the engine's fp32 mode is within 2x the reference's own fp32-vs-fp64
  error of the fp64 twin, and the bf16 mode's error is of the order of the
  reference's bf16-weight sensitivity.
* bf16 at full length, both configs: bitwise determinism, loss ~ log V (the
  reference's known answer for near-uniform predictions,
  pkg/tests/test_training.py:36-41) and the update w - fp32(lr*scale)*g with a
  forced clip (training.py:123-142).
"""

import math

import numpy as np
import pytest

from oracle import minmt_oracle as O
from tests.gpu_helpers import step_close

pytestmark = pytest.mark.gpu

WIDTH = {"c3": (50000, 1024, 1024, 4, 128), "c5": (100000, 1024, 1024, 2, 256)}
FULL_LEN = {"c3": 50, "c5": 80}
FP32_TOL, BF16_TOL = 1e-4, 2e-2


def _setup(name, n):
    from paper_1802_07170_b200.model import Batch, Model, ModelConfig, Rng
    V, E, H, L, B = WIDTH[name]
    cfg = ModelConfig(V, E, H, L, 0.2)
    params = {b.name: b.var.data.copy() for b in Model.new(cfg, Rng(1)).params.blocks()}
    src, sm, tgt, tm = O.synthetic_batch(V, n, n, B, seed=2, ragged=True)
    return cfg, O.Dims(V, E, H, L, 0.2), params, (src, sm, tgt, tm), Batch(src, tgt, sm, tm)


def _engine(cfg, mode, params):
    from paper_1802_07170_b200.engine import Engine
    eng = Engine(cfg, mode=mode)
    eng.upload(params)
    return eng


@pytest.mark.parametrize("name", list(WIDTH))
def test_fullwidth_step_matches_oracle(name):
    cfg, d, params, raw, batch = _setup(name, 8)
    names = [n for n, _ in O.registry(d)]
    gen_ref = np.random.Generator(np.random.PCG64(5))
    p_ref = {k: v.copy() for k, v in params.items()}
    ol, og, _ = O.forward_backward(p_ref, d, *raw, 0.1, gen=gen_ref)
    lr, clip = 1.0, 0.5  # the clip binds (norm ~1 at init): scale = clip / norm is exercised
    onorm = O.sgd_step(p_ref, og, names, lr, clip)
    assert onorm > clip
    for mode, tol in (("fp32", FP32_TOL), ("bf16", BF16_TOL)):
        eng = _engine(cfg, mode, params)
        gen = np.random.Generator(np.random.PCG64(5))
        loss, _ = eng.step(batch, lr, clip, 0.1, gen, update=False)
        grads = eng.grads()
        assert abs(loss - ol) <= tol * abs(ol), (mode, loss, ol)
        errs = {n: O.norm_rel_err(grads[n], og[n]) for n in names}
        assert max(errs.values()) < tol, (mode, sorted(errs.items(), key=lambda x: -x[1])[:5])
        assert gen.bit_generator.state == gen_ref.bit_generator.state, mode
        eng.close()
        eng = _engine(cfg, mode, params)
        _, norm = eng.step(batch, lr, clip, 0.1, np.random.Generator(np.random.PCG64(5)))
        newp = eng.params()
        eng.close()
        assert abs(norm - onorm) <= tol * onorm, (mode, norm, onorm)
        errs = {n: O.norm_rel_err(newp[n], p_ref[n]) for n in names}
        assert max(errs.values()) < tol, (mode, sorted(errs.items(), key=lambda x: -x[1])[:5])
        # the applied step itself (w_new - w_old) against the reference's step,
        # floored at a few fp32 ulps of the weights (w - s*g rounds to fp32)
        rel = 1e-3 if mode == "fp32" else 5 * BF16_TOL
        for n in names:
            ok, err = step_close(newp[n], params[n], p_ref[n], rel)
            assert ok, (mode, n, err)


def test_full_length_c3_within_reference_floor():
    cfg, d, params, raw, batch = _setup("c3", FULL_LEN["c3"])
    ol, og, _ = O.forward_backward({k: v.copy() for k, v in params.items()}, d, *raw, 0.1,
                                   gen=np.random.Generator(np.random.PCG64(5)))
    l64, g64, _ = O.forward_backward({k: v.astype(np.float64) for k, v in params.items()}, d, *raw, 0.1,
                                     gen=np.random.Generator(np.random.PCG64(5)))
    floor = max(O.norm_rel_err(og[n], g64[n]) for n in og)  # the reference's own fp32 error
    res = {}
    for mode in ("fp32", "bf16"):
        eng = _engine(cfg, mode, params)
        loss, _ = eng.step(batch, 1.0, 5.0, 0.1, np.random.Generator(np.random.PCG64(5)), update=False)
        res[mode] = (loss, eng.grads())
        eng.close()
    loss32, g32 = res["fp32"]
    assert abs(loss32 - l64) <= FP32_TOL * abs(l64)
    err32 = max(O.norm_rel_err(g32[n], g64[n]) for n in og)
    assert err32 <= 2 * floor, (err32, floor)
    # bf16: the loss to 2e-2; the gradients within the trajectory sensitivity the
    # reference itself shows when only its weights are stored in bf16
    import torch
    pw = {k: torch.from_numpy(v).to(torch.bfloat16).float().numpy() for k, v in params.items()}
    _, gw, _ = O.forward_backward(pw, d, *raw, 0.1, gen=np.random.Generator(np.random.PCG64(5)))
    sens = max(O.norm_rel_err(gw[n], og[n]) for n in og)
    loss16, g16 = res["bf16"]
    assert abs(loss16 - ol) <= BF16_TOL * abs(ol)
    err16 = max(O.norm_rel_err(g16[n], og[n]) for n in og)
    assert err16 <= 2 * sens, (err16, sens)


@pytest.mark.parametrize("name", list(WIDTH))
def test_full_length_bf16_properties(name):
    cfg, d, params, raw, batch = _setup(name, FULL_LEN[name])
    V, L = d.vocab, d.depth
    runs = []
    for _ in range(2):
        eng = _engine(cfg, "bf16", params)
        gen = np.random.Generator(np.random.PCG64(5))
        loss, _ = eng.step(batch, 1.0, 5.0, 0.1, gen, update=False)
        runs.append((loss, eng.grads(), gen.bit_generator.state))
        eng.close()
    (l1, g1, s1), (l2, g2, s2) = runs
    assert l1 == l2 and s1 == s2
    for n in g1:
        assert np.array_equal(g1[n], g2[n]), n
    assert abs(l1 - math.log(V)) < 0.02 * math.log(V), (l1, math.log(V))
    lr, clip = 0.5, 0.05  # a small clip so the scale is exercised
    eng = _engine(cfg, "bf16", params)
    _, norm = eng.step(batch, lr, clip, 0.1, np.random.Generator(np.random.PCG64(5)))
    w1 = eng.params()
    eng.close()
    gnorm = math.sqrt(sum(float(np.dot(g.ravel().astype(np.float64), g.ravel().astype(np.float64)))
                          for g in g1.values()))
    assert abs(norm - gnorm) <= 1e-3 * gnorm
    s32 = np.float32(lr * min(1.0, clip / norm))
    for n in ("out.w", "att.w_c.w", f"dec.l{L}.w_i", "src_embed"):
        exp = params[n] - s32 * g1[n]
        assert O.norm_rel_err(w1[n] - params[n], exp - params[n]) < 1e-5, n
