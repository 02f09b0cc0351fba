"""Bit-exact masking / indexing and the train-step API semantics on the device.

* masked attention weights are exactly 0.0 and every column sums to 1
  (pkg/tests/test_attention.py:61-71); masked source positions receive exactly
  zero gradient from attention (pkg/tests/test_attention.py:181-190);
* gathered embedding rows equal the table rows bit for bit, and the shifted
  decoder input is BOS then tgt[:-1] (tensor.py:191-205, model.py:239-244);
* ParamBlock.learnable=False blocks are left out of the norm and the update
  (training.py:128-139, pkg/tests/test_training.py:121-125);
* clip_norm=0.0 clips to a zero step (training.py:136-137: the reference clips
  whenever clip_norm is not None and norm > clip_norm);
* a Trainer-like sequence (step, copy_data, steps, load_data(best), step) in
  eager mode trains from the restored weights (training.py:246-254).
"""

import numpy as np
import pytest

from oracle import minmt_oracle as O
from tests.gpu_helpers import cfg_of, oracle_step, scaled_params, step_close

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
@pytest.mark.parametrize("L", [1, 2])
def test_masked_attention_exact_zeros(mode, L):
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    V, E, H, B, S, T = 256, 64, 256, 12, 11, 9
    d = O.Dims(V, E, H, L, 0.0)
    params = scaled_params(d, 3, 0.1)
    src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=5, ragged=True)
    eng = Engine(cfg_of(d), mode=mode)
    eng.upload(params)
    eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, None, update=False)
    alpha = eng.debug_buffer("alpha").reshape(B, T, S)  # [b][t][s]
    dhs = eng.debug_buffer("dtop" if L == 1 else f"dy:{L}").reshape(S, B, H)  # d(top encoder output)
    eng.close()
    masked = sm.T[:, None, :] == 0  # (B, 1, S)
    assert (alpha[np.broadcast_to(masked, alpha.shape)] == 0.0).all()
    assert (alpha[np.broadcast_to(~masked, alpha.shape)] > 0.0).all()
    assert np.allclose(alpha.sum(axis=2), 1.0, atol=1e-5)
    pad = sm == 0  # (S, B)
    assert not dhs[pad].any()
    assert dhs[~pad].any(axis=-1).all()


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_embedding_gather_bit_exact(mode):
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    V, E, H, B, S, T = 304, 64, 256, 8, 7, 6
    d = O.Dims(V, E, H, 1, 0.0)
    params = scaled_params(d, 4, 0.1)
    src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=6, ragged=True)
    eng = Engine(cfg_of(d), mode=mode)
    eng.upload(params)
    eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, None, update=False)
    xs = eng.debug_buffer("Xs").reshape(S * B, E)
    xt = eng.debug_buffer("Xt").reshape(T * B, E)
    eng.close()

    def stored(a):  # the table as the engine stores the activation (bf16 in production mode)
        if mode == "fp32":
            return a
        import torch
        return torch.from_numpy(a).to(torch.bfloat16).float().numpy()
    assert np.array_equal(xs, stored(params["src_embed"])[src.reshape(-1)])
    tin = O.shift_targets(tgt)
    assert (tin[0] == 2).all() and np.array_equal(tin[1:], tgt[:-1])
    assert np.array_equal(xt, stored(params["tgt_embed"])[tin.reshape(-1)])


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_learnable_false_blocks_frozen(mode):
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    d = O.Dims(96, 32, 256, 2, 0.0)
    params = scaled_params(d, 2, 0.1)
    batch = O.synthetic_batch(96, 7, 6, 8, seed=2, ragged=True)
    frozen = {"src_embed", "enc.l1.fwd.w_f", "dec.l2.b_o", "att.w_c.w"}
    names = [n for n, _ in O.registry(d)]
    # oracle: norm and update over the learnable blocks only (training.py:128-139)
    p = {k: v.copy() for k, v in params.items()}
    _, g, _ = O.forward_backward(p, d, *batch, 0.1)
    onorm = O.sgd_step(p, g, [n for n in names if n not in frozen], 1.0, 0.05)
    tol = 1e-4 if mode == "fp32" else 2e-2
    eng = Engine(cfg_of(d), mode=mode)
    eng.upload(params)
    eng.set_learnable({n: n not in frozen for n in names})
    src, sm, tgt, tm = batch
    _, norm = eng.step(Batch(src, tgt, sm, tm), 1.0, 0.05, 0.1, None)
    newp = eng.params()
    eng.close()
    assert abs(norm - onorm) <= tol * onorm
    for n in names:
        if n in frozen:
            assert np.array_equal(newp[n], params[n]), n
        else:
            assert step_close(newp[n], params[n], p[n], 1e-3 if mode == "fp32" else 0.1)[0], n


def test_zero_clip_norm_is_a_zero_step():
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    d = O.Dims(96, 32, 256, 1, 0.0)
    params = scaled_params(d, 2, 0.1)
    src, sm, tgt, tm = O.synthetic_batch(96, 5, 6, 8, seed=2)
    eng = Engine(cfg_of(d), mode="fp32")
    eng.upload(params)
    _, norm = eng.step(Batch(src, tgt, sm, tm), 1.0, 0.0, 0.1, None)
    newp = eng.params()
    eng.close()
    assert norm > 0
    for n in params:
        assert np.array_equal(newp[n], params[n]), n


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_trainer_restore_from_best_eager(mode):
    """The reference Trainer's restore-from-best (training.py:205, 246-254):
    best = copy_data(); more steps; load_data(best); next step trains from best.
    In eager mode (host mirrors device) the restore must reach the device."""
    from paper_1802_07170_b200 import training as TR
    from paper_1802_07170_b200.model import Batch, Model, ModelConfig, ModelParams, Rng, TrainConfig
    saved = (ModelParams.copy_data, ModelParams.load_data, dict(TR.DEFAULTS))
    try:
        TR.DEFAULTS["sync"] = "eager"
        cfg = ModelConfig(96, 32, 256, 2, 0.0)
        d = O.Dims(96, 32, 256, 2, 0.0)
        model = Model.new(cfg, Rng(1))
        src, sm, tgt, tm = O.synthetic_batch(96, 7, 6, 8, seed=2, ragged=True)
        batch, tcfg = Batch(src, tgt, sm, tm), TrainConfig()
        TR.train_step(model, batch, tcfg, 1.0, Rng(5), mode=mode)
        best = model.params.copy_data()
        assert isinstance(best, dict)
        for _ in range(2):
            TR.train_step(model, batch, tcfg, 1.0, Rng(5), mode=mode)
        model.params.load_data(best)
        TR.train_step(model, batch, tcfg, 1.0, Rng(5), mode=mode)
        got = {b.name: b.var.data for b in model.params.blocks()}
        ol, onorm, _, op, _ = oracle_step(d, best, (src, sm, tgt, tm), 0.1, 1.0, 5.0, 5, update=True)
        tol = 1e-4 if mode == "fp32" else 2e-2
        for n in op:
            assert step_close(got[n], best[n], op[n], 1e-3 if mode == "fp32" else 0.1)[0], n
            assert O.norm_rel_err(got[n], op[n]) < tol, n
    finally:
        ModelParams.copy_data, ModelParams.load_data = saved[0], saved[1]
        ModelParams._cmt_patched = False
        TR.DEFAULTS.clear()
        TR.DEFAULTS.update(saved[2])


def test_nonfinite_norm_leaves_grads_like_reference():
    """training.py:133-134: a non-finite norm raises before the grads are zeroed."""
    from paper_1802_07170_b200 import training as TR
    from paper_1802_07170_b200.errors import NumericError
    from paper_1802_07170_b200.model import Batch, Model, ModelConfig, Rng, TrainConfig
    model = Model.new(ModelConfig(96, 32, 256, 1, 0.0), Rng(1))
    blk = {b.name: b for b in model.params.blocks()}
    blk["att.w_a.w"].var.data[0, 0] = np.float32(3e38)  # overflows the grad norm only
    src, sm, tgt, tm = O.synthetic_batch(96, 5, 6, 8, seed=2)
    before = {n: b.var.data.copy() for n, b in blk.items()}
    try:
        TR.train_step(model, Batch(src, tgt, sm, tm), TrainConfig(), 1.0, Rng(5), mode="fp32", sync="eager")
    except NumericError as e:
        assert "gradient norm" in str(e), str(e)
    else:
        pytest.skip("this perturbation kept the norm finite")
    for n, b in blk.items():
        assert np.array_equal(b.var.data, before[n]), n
    assert any(b.var.grad.any() for b in blk.values())


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_c_abi_train_step_matches_engine_step(mode):
    """cmt_train_step, the reference-facing C entry point (host ids/masks in,
    loss out; include/cytonmt_b200.h), called through ctypes exactly as the
    INTEGRATION.md binding does, equals Engine.step (stage + run) bit for bit,
    and advances the caller's PCG64 state by the reported draws -- including
    the calls that capture and replay the step graph."""
    import ctypes

    from paper_1802_07170_b200 import _lib
    from paper_1802_07170_b200.engine import Engine, pcg_state
    from paper_1802_07170_b200.model import Batch
    d = O.Dims(96, 32, 256, 2, 0.2)
    params = scaled_params(d, 6, 0.1)
    # three batches of one shape: the ABI engine captures its step graph on the
    # second call and replays it on the third; the reference engine stays eager
    batches = [O.synthetic_batch(96, 7, 6, 8, seed=3 + i, ragged=True) for i in range(3)]
    out = []
    for via_abi in (False, True):
        eng = Engine(cfg_of(d), mode=mode)
        if not via_abi:
            eng.set_option("graph", 0)
        eng.upload(params)
        gen = np.random.Generator(np.random.PCG64(11))
        losses = []
        for src, sm, tgt, tm in batches:
            if via_abi:
                s, sm_, t, tm_ = (np.ascontiguousarray(x) for x in (src.astype(np.int64), sm.astype(np.float32),
                                                                     tgt.astype(np.int64), tm.astype(np.float32)))
                st = pcg_state(gen)
                args = _lib.StepArgs(1.0, 0.5, 0.1, st[0], st[1], st[2], st[3], 0.0, 0)
                res = _lib.StepResult()
                llp, fp = ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_float)
                rc = eng.lib.cmt_train_step(eng.h, s.ctypes.data_as(llp), sm_.ctypes.data_as(fp), s.shape[0],
                                            t.ctypes.data_as(llp), tm_.ctypes.data_as(fp), t.shape[0], s.shape[1],
                                            ctypes.byref(args), ctypes.byref(res))
                assert rc == 0, eng.lib.cmt_last_error(eng.h)
                gen.bit_generator.advance(int(res.draws))
                losses.append((res.loss, res.grad_norm))
            else:
                losses.append(eng.step(Batch(src, tgt, sm, tm), 1.0, 0.5, 0.1, gen))
        replays = eng.stat("graph_replays")[0]
        out.append((losses, eng.params(), gen.bit_generator.state, replays))
        eng.close()
    assert out[0][3] == 0 and out[1][3] == 2
    assert out[0][0] == out[1][0] and out[0][2] == out[1][2]
    for n in out[0][1]:
        assert np.array_equal(out[0][1][n], out[1][1][n]), n
