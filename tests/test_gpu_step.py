"""Whole-step GPU parity through the C ABI.

* fp32 validation mode vs the REFERENCE's own outputs (golden fixtures from
  tests/golden/make_golden.py): loss, every per-block gradient, the updated
  weights, the gradient norm and the dropout RNG state, at 1e-4 norm-relative
  (the north-star fp32 tolerance; metric of pkg/tests/helpers.py:80-81).
* bf16 production mode vs the oracle at 2e-2 norm-relative.
* error semantics: ConfigError / MaskError / NumericError with weights unchanged.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import minmt_oracle as O  # noqa: E402
from tests.gpu_helpers import engine_step, oracle_step, scaled_params  # noqa: E402

GOLDEN = ["toy", "toy_dropout", "ragged_clip", "notanh_shared", "deep_noclip"]
FP32_TOL = 1e-4
BF16_TOL = 2e-2


def update_err(new, init, ref_new, ulps=4):
    """Error of the applied step (w_new - w_old) relative to the reference step
    size, floored at a few fp32 ulps of the weights (w - lr*g rounds to fp32)."""
    new, init, ref_new = (np.asarray(x, np.float64) for x in (new, init, ref_new))
    ulp = float(np.spacing(np.float32(np.abs(ref_new).max())))
    return float(np.abs(new - ref_new).max() / (np.abs(ref_new - init).max() + ulps * ulp + 1e-30))


def dims_of(g):
    return O.Dims(int(g["V"]), int(g["E"]), int(g["H"]), int(g["L"]), float(g["dropout"]), bool(g["tanh"]),
                  bool(g["shared"]))


def golden_args(g):
    clip = None if float(g["clip"]) < 0 else float(g["clip"])
    batch = (g["src"], g["src_mask"], g["tgt"], g["tgt_mask"])
    return batch, float(g["eps"]), float(g["lr"]), clip, int(g["seed"]) + 5


@pytest.mark.parametrize("case", GOLDEN)
def test_fp32_step_matches_reference_golden(golden, case):
    g = golden(case)
    d = dims_of(g)
    names = [str(n) for n in g["names"]]
    params = {n: g[f"init:{n}"] for n in names}
    batch, eps, lr, clip, seed = golden_args(g)
    # grads (no update)
    loss, _, grads, _, _ = engine_step(d, params, batch, eps, lr, clip, seed, "fp32", update=False)
    assert abs(loss - float(g["loss"])) <= FP32_TOL * abs(float(g["loss"]))
    for n in names:
        assert O.norm_rel_err(grads[n], g[f"grad:{n}"]) < FP32_TOL, n
    # full step: norm, updated weights, RNG state
    loss, norm, _, newp, gen = engine_step(d, params, batch, eps, lr, clip, seed, "fp32", update=True)
    assert abs(norm - float(g["norm"])) <= FP32_TOL * float(g["norm"])
    errs = {n: O.norm_rel_err(newp[n], g[f"new:{n}"]) for n in names}
    assert max(errs.values()) < FP32_TOL, errs
    # the step itself (w_new - w_old) to 1e-3 of its size, floored at a few fp32 ulps
    errs = {n: update_err(newp[n], g[f"init:{n}"], g[f"new:{n}"]) for n in names}
    assert max(errs.values()) < 1e-3, errs
    st = gen.bit_generator.state["state"]
    ref = [int(x) for x in g["rng_state"]]
    assert (st["state"] >> 64, st["state"] & ((1 << 64) - 1)) == (ref[0], ref[1])


def test_fp32_tiny_config_checksums(golden):
    """BASELINE configs[0] (V=1k, H=128, B=16, len 20) against reference checksums."""
    from paper_1802_07170_b200.model import Model, ModelConfig, Rng
    g = golden("tiny")
    d = dims_of(g)
    m = Model.new(ModelConfig(d.vocab, d.emb, d.hidden, d.depth, d.dropout), Rng(int(g["seed"])))
    params = {b.name: b.var.data for b in m.params.blocks()}
    batch, eps, lr, clip, seed = golden_args(g)
    loss, _, grads, _, _ = engine_step(d, params, batch, eps, lr, clip, seed, "fp32", update=False)
    assert abs(loss - float(g["loss"])) <= FP32_TOL * float(g["loss"])
    for n, gr in grads.items():
        ck = g[f"grad:{n}"]
        gg = gr.astype(np.float64).ravel()
        idx = np.linspace(0, gg.size - 1, num=min(16, gg.size)).astype(np.int64)
        scale = max(np.abs(gg).max(), 1e-30)
        assert abs(np.sqrt((gg * gg).sum()) - np.sqrt(ck[1])) <= FP32_TOL * np.sqrt(ck[1]) + 1e-12, n
        assert np.abs(gg[idx] - ck[4:4 + idx.size]).max() <= FP32_TOL * scale, n


BF16_CASES = {
    # (V, E, H, L, B, S, T, dropout, tanh, shared, ragged, eps, clip)
    "small_ragged": (64, 32, 32, 2, 8, 7, 6, 0.2, True, False, True, 0.1, 5.0),
    "deep_shared_clip": (96, 16, 24, 3, 6, 5, 9, 0.1, True, True, True, 0.1, 0.02),
    "notanh_b1": (40, 64, 64, 2, 1, 6, 5, 0.0, False, False, False, 0.0, None),
    "tiny_cfg": (1000, 128, 128, 1, 16, 20, 20, 0.2, True, False, True, 0.1, 5.0),
}


@pytest.mark.parametrize("case", list(BF16_CASES))
def test_bf16_step_matches_oracle(case):
    V, E, H, L, B, S, T, p, tanh_, shared, ragged, eps, clip = BF16_CASES[case]
    d = O.Dims(V, E, H, L, p, tanh_, shared)
    params = scaled_params(d, 3, 0.1)
    batch = O.synthetic_batch(V, S, T, B, seed=4, ragged=ragged)
    lr, seed = 1.0, 21
    ol, _, og, _, ogen = oracle_step(d, params, batch, eps, lr, clip, seed, update=False)
    loss, _, grads, _, gen = engine_step(d, params, batch, eps, lr, clip, seed, "bf16", update=False)
    assert abs(loss - ol) <= BF16_TOL * abs(ol)
    errs = {n: O.norm_rel_err(grads[n], og[n]) for n in grads}
    assert max(errs.values()) < BF16_TOL, {n: e for n, e in errs.items() if e >= BF16_TOL}
    assert gen.bit_generator.state == ogen.bit_generator.state
    # updated weights (delta) vs the oracle's update
    ol, onorm, _, op, _ = oracle_step(d, params, batch, eps, lr, clip, seed, update=True)
    loss, norm, _, newp, _ = engine_step(d, params, batch, eps, lr, clip, seed, "bf16", update=True)
    assert abs(norm - onorm) <= BF16_TOL * onorm
    errs = {n: O.norm_rel_err(newp[n], op[n]) for n in newp}
    assert max(errs.values()) < BF16_TOL, {n: e for n, e in errs.items() if e >= BF16_TOL}
    errs = {n: update_err(newp[n], params[n], op[n], ulps=64) for n in newp}
    assert max(errs.values()) < 5 * BF16_TOL, {n: e for n, e in errs.items() if e >= 5 * BF16_TOL}


@pytest.mark.slow
def test_bf16_c2_config_matches_oracle():
    """BASELINE configs[1]: 2-layer bi-enc 512, V=30k, B=64, len 50 (oracle ~6 s)."""
    d = O.Dims(30000, 512, 512, 2, 0.2)
    params = scaled_params(d, 5, 0.1)
    batch = O.synthetic_batch(30000, 50, 50, 64, seed=0, ragged=True)
    ol, _, og, _, _ = oracle_step(d, params, batch, 0.1, 1.0, 5.0, 5, update=False)
    loss, _, grads, _, _ = engine_step(d, params, batch, 0.1, 1.0, 5.0, 5, "bf16", update=False)
    assert abs(loss - ol) <= BF16_TOL * ol
    worst = max(O.norm_rel_err(grads[n], og[n]) for n in grads)
    assert worst < BF16_TOL, worst


def test_fp32_c2_shape_matches_oracle_small_vocab():
    d = O.Dims(512, 64, 64, 2, 0.2)
    params = scaled_params(d, 8, 0.1)
    batch = O.synthetic_batch(512, 30, 25, 32, seed=2, ragged=True)
    ol, _, og, _, _ = oracle_step(d, params, batch, 0.1, 1.0, 5.0, 9, update=False)
    loss, _, grads, _, _ = engine_step(d, params, batch, 0.1, 1.0, 5.0, 9, "fp32", update=False)
    assert abs(loss - ol) <= FP32_TOL * ol
    for n in grads:
        assert O.norm_rel_err(grads[n], og[n]) < FP32_TOL, n


# ---- error semantics ----

def _small():
    d = O.Dims(64, 16, 16, 2, 0.2)
    return d, scaled_params(d, 1, 0.1), O.synthetic_batch(64, 5, 4, 4, seed=1)


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_bad_token_id_raises_config_error(mode):
    from paper_1802_07170_b200.errors import ConfigError
    d, params, (src, sm, tgt, tm) = _small()
    src = src.copy()
    src[2, 1] = 64
    with pytest.raises(ConfigError, match="token id 64 outside vocabulary of size 64"):
        engine_step(d, params, (src, sm, tgt, tm), 0.1, 1.0, 5.0, 1, mode)


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_fully_masked_column_raises_mask_error(mode):
    from paper_1802_07170_b200.errors import MaskError
    d, params, (src, sm, tgt, tm) = _small()
    sm = sm.copy()
    sm[:, 2] = 0
    with pytest.raises(MaskError):
        engine_step(d, params, (src, sm, tgt, tm), 0.1, 1.0, 5.0, 1, mode)


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_nonfinite_aborts_without_update(mode):
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.errors import NumericError
    from paper_1802_07170_b200.model import Batch
    from tests.gpu_helpers import cfg_of
    d, params, (src, sm, tgt, tm) = _small()
    params = {k: v.copy() for k, v in params.items()}
    params["out.w"][5, 3] = np.nan     # logits column 3 non-finite -> NumericError, nothing moves
    eng = Engine(cfg_of(d), mode=mode)
    eng.upload(params)
    with pytest.raises(NumericError):
        eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, np.random.default_rng(0))
    after = eng.params()
    for n in params:
        assert np.array_equal(after[n], params[n], equal_nan=True), n


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_drop_in_train_step_and_determinism(mode):
    """training.train_step on the host mirror: reference semantics (loss float,
    params updated, grads zero, rng advanced); two identical runs are bit-identical."""
    from paper_1802_07170_b200 import training
    from paper_1802_07170_b200.model import Batch, Model, ModelConfig, Rng, TrainConfig
    outs = []
    for _ in range(2):
        m = Model.new(ModelConfig(80, 32, 32, 2, 0.2), Rng(3))
        src, sm, tgt, tm = O.synthetic_batch(80, 6, 5, 8, seed=3, ragged=True)
        rng = Rng(7)
        losses = [training.train_step(m, Batch(src, tgt, sm, tm), TrainConfig(), 1.0, rng, mode=mode)
                  for _ in range(3)]
        assert all(isinstance(x, float) for x in losses) and losses[2] < losses[0]
        assert all(not b.var.grad.any() for b in m.params.blocks())
        outs.append((losses, {b.name: b.var.data.copy() for b in m.params.blocks()}, rng.gen.random()))
    assert outs[0][0] == outs[1][0] and outs[0][2] == outs[1][2]
    for n in outs[0][1]:
        assert np.array_equal(outs[0][1][n], outs[1][1][n]), n


@pytest.mark.parametrize("case", [(256, 128, 256, 2, 32, 11, 9, True), (512, 64, 256, 3, 128, 7, 12, True),
                                  (304, 64, 512, 1, 5, 13, 4, False), (256, 256, 256, 2, 96, 6, 5, True),
                                  (256, 64, 1024, 1, 256, 5, 4, True)])  # B=256: 128-row slices, two per scan
def test_persistent_recurrence_matches_per_step_and_oracle(case):
    """The persistent recurrent kernels (default in bf16) against the per-step
    tcgen05 path and the oracle, masked + unmasked, forward + reverse scans,
    partial batch slices (B not a multiple of the slice rows)."""
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    from tests.gpu_helpers import cfg_of
    V, E, H, L, B, S, T, ragged = case
    d = O.Dims(V, E, H, L, 0.2)
    params = scaled_params(d, 11, 0.1)
    src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=6, ragged=ragged)
    _, _, og, _, _ = oracle_step(d, params, (src, sm, tgt, tm), 0.1, 1.0, 5.0, 3, update=False)
    out = {}
    variants = {  # option settings per variant ("dual" = the default configuration)
        "per_step": dict(persistent=0, dual=0),  # one tcgen05 GEMM per step, cell in the epilogue
        "single": dict(dual=0),  # every scan alone: lstm_fwd_multi<64|128> / lstm_bwd_multi<64|128>
        "dual": dict(),  # default: paired forward scans in lstm_fwd_tm, paired BPTT in lstm_bwd_multi<128>
        "dual_multi": dict(fwd_tm=0),  # paired forward scans in lstm_fwd_multi<128>
        "no_bg": dict(bwd_bg=0),  # every BPTT weight-gradient column on the main streams
    }
    for variant, opts in variants.items():
        eng = Engine(cfg_of(d), mode="bf16")
        for k, v in opts.items():
            eng.set_option(k, v)
        eng.upload(params)
        eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, np.random.Generator(np.random.PCG64(3)), update=False)
        out[variant] = eng.grads()
        eng.close()
    for v in ("single", "dual", "dual_multi", "no_bg"):
        for n in og:
            assert O.norm_rel_err(out[v][n], out["per_step"][n]) < BF16_TOL, (v, n)
            assert O.norm_rel_err(out[v][n], og[n]) < BF16_TOL, (v, n)


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_dp_path_single_rank_nccl_matches_plain(mode):
    """The data-parallel branch (NCCL all-reduce of grads/loss/status, dense
    embedding grads, union-of-rows update) on a 1-rank communicator equals the
    plain single-GPU step."""
    from paper_1802_07170_b200 import dp
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    from tests.gpu_helpers import cfg_of
    d = O.Dims(96, 32, 256, 2, 0.0)
    params = scaled_params(d, 2, 0.1)
    src, sm, tgt, tm = O.synthetic_batch(96, 7, 6, 8, seed=2, ragged=True)
    out = []
    for use_dp, ar_overlap in ((False, 1), (True, 1), (True, 0)):
        eng = Engine(cfg_of(d), mode=mode)
        eng.set_option("ar_overlap", ar_overlap)  # bucketed all-reduce on the comm stream during the backward
        eng.upload(params)
        if use_dp:
            dp.attach(eng, None, 0, 1)
        loss, norm = eng.step(Batch(src, tgt, sm, tm), 1.0, 0.05, 0.1, None)
        out.append((loss, norm, eng.params()))
        eng.close()
    for k in (1, 2):
        assert abs(out[0][0] - out[k][0]) <= 1e-6 * abs(out[0][0])
        assert abs(out[0][1] - out[k][1]) <= 1e-5 * out[0][1]
        for n in out[0][2]:
            assert O.norm_rel_err(out[k][2][n], out[0][2][n]) < 1e-6, n


@pytest.mark.parametrize("case", [(304, 64, 128, 2, 24, 17, 13, True), (256, 128, 256, 1, 8, 64, 64, False),
                                  (256, 64, 128, 1, 12, 80, 72, True), (256, 64, 128, 1, 4, 128, 100, False),
                                  (256, 64, 128, 1, 3, 200, 150, True)])
def test_attention_variants_agree(case):
    """The tcgen05 attention core (batched per-sentence GEMMs + softmax
    kernels, the bf16 default for S <= 256) against the SIMT kernels (split
    many-CTA, per-sentence tiled) and the oracle (bf16 step)."""
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    from tests.gpu_helpers import cfg_of
    V, E, H, L, B, S, T, ragged = case
    d = O.Dims(V, E, H, L, 0.0)
    params = scaled_params(d, 13, 0.1)
    src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=8, ragged=ragged)
    _, _, og, _, _ = oracle_step(d, params, (src, sm, tgt, tm), 0.1, 1.0, 5.0, 3, update=False)
    out = {}
    variants = {"tc": dict(), "split2": dict(att_tc=0, att_split=2), "split1": dict(att_tc=0, att_split=1),
                "tiled": dict(att_tc=0, att_split=0)}
    if S > 128:  # beyond the SIMT kernels' tiles: the tcgen05 core alone against the oracle
        variants = {"tc": dict()}
    for name, opts in variants.items():
        eng = Engine(cfg_of(d), mode="bf16")
        for k, v in opts.items():
            eng.set_option(k, v)
        eng.upload(params)
        eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, np.random.Generator(np.random.PCG64(3)), update=False)
        out[name] = eng.grads()
        eng.close()
    for v in variants:
        for n in og:
            assert O.norm_rel_err(out[v][n], og[n]) < BF16_TOL, (v, n)
            if v != "tc":
                assert O.norm_rel_err(out[v][n], out["split2" if v != "split2" else "tiled"][n]) < 1e-3, (v, n)


@pytest.mark.parametrize("mode,tol", [("fp32", FP32_TOL), ("bf16", BF16_TOL)])
@pytest.mark.parametrize("case", GOLDEN)
def test_dev_entropy_matches_reference_golden(golden, case, mode, tol):
    """INFER-mode device forward (dev_entropy, training.py:162-182) against the
    reference's own value (tests/golden/make_dev_golden.py); dropout draws none."""
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    from tests.gpu_helpers import cfg_of
    g = golden(case)
    dv = golden("dev_entropy")
    d = dims_of(g)
    if mode == "bf16" and any(x % 8 for x in (d.vocab, d.emb, d.hidden)):
        pytest.skip("bf16 mode needs dims that are multiples of 8")
    names = [str(n) for n in g["names"]]
    eng = Engine(cfg_of(d), mode=mode)
    eng.upload({n: g[f"init:{n}"] for n in names})
    batches = [Batch(g["src"], g["tgt"], g["src_mask"], g["tgt_mask"]),
               Batch(dv[f"{case}:src2"], dv[f"{case}:tgt2"], dv[f"{case}:sm2"], dv[f"{case}:tm2"])]
    val = eng.dev_entropy(batches)
    ref = float(dv[f"{case}:value"])
    assert abs(val - ref) <= tol * abs(ref), (val, ref)
    # the pass left the weights alone
    newp = eng.params()
    for n in names:
        assert np.array_equal(newp[n], g[f"init:{n}"].astype(np.float32)), n
    eng.close()


def test_dev_entropy_drop_in_and_empty_batch():
    """training.dev_entropy (drop-in signature) = oracle on a c-tiny-like model;
    a batch with no unmasked target contributes nothing; empty list raises."""
    from paper_1802_07170_b200 import training
    from paper_1802_07170_b200.errors import ConfigError
    from paper_1802_07170_b200.model import Batch, Model, ModelConfig, Rng
    cfg = ModelConfig(256, 64, 256, 2, 0.2)
    model = Model.new(cfg, Rng(4))
    d = O.Dims(256, 64, 256, 2, 0.2)
    b1 = O.synthetic_batch(256, 9, 7, 16, seed=2, ragged=True)
    b2 = O.synthetic_batch(256, 5, 11, 16, seed=3, ragged=False)
    params = {b.name: b.var.data.copy() for b in model.params.blocks()}
    ref = O.dev_entropy(params, d, [b1, b2])
    src, sm, tgt, tm = b2
    empty = Batch(src, tgt, sm, np.zeros_like(tm))
    batches = [Batch(b1[0], b1[2], b1[1], b1[3]), Batch(src, tgt, sm, tm), empty]
    val = training.dev_entropy(model, batches, mode="bf16")
    assert abs(val - ref) <= BF16_TOL * ref, (val, ref)
    with pytest.raises(ConfigError):
        training.dev_entropy(model, [], mode="bf16")


@pytest.mark.gpu
def test_device_snapshot_and_restore_from_best():
    """ModelParams.copy_data / load_data through install(sync="lazy"): the
    snapshot stays on the device (a read-only name -> array mapping equal to the
    parameters at that point), load_data restores it device-to-device exactly,
    and a plain host dict still round-trips (model.py:104-115, training.py:246-254)."""
    import types

    from paper_1802_07170_b200 import training as TR
    from paper_1802_07170_b200.engine import DeviceSnapshot
    from paper_1802_07170_b200.model import Batch, Model, ModelConfig, ModelParams, Rng, TrainConfig
    saved = (ModelParams.copy_data, ModelParams.load_data, dict(TR.DEFAULTS))
    fake = types.SimpleNamespace(train_step=None, dev_entropy=None, save_checkpoint=lambda path, model, vocab: None)
    try:
        TR.install(fake, sync="lazy", params_cls=ModelParams)
        cfg = ModelConfig(96, 32, 256, 2, 0.2)
        model = Model.new(cfg, Rng(1))
        src, sm, tgt, tm = O.synthetic_batch(96, 7, 6, 8, seed=2, ragged=True)
        batch, tcfg, rng = Batch(src, tgt, sm, tm), TrainConfig(), Rng(5)
        fake.train_step(model, batch, tcfg, 1.0, rng)
        snap = model.params.copy_data()
        assert isinstance(snap, DeviceSnapshot) and list(snap) == [b.name for b in model.params.blocks()]
        TR.sync_to_host(model)
        ref = {b.name: b.var.data.copy() for b in model.params.blocks()}
        for n in ref:
            assert np.array_equal(snap[n], ref[n]), n
        for _ in range(2):
            fake.train_step(model, batch, tcfg, 1.0, rng)
        eng = TR.engine_for(model)
        moved = eng.params()
        assert any(not np.array_equal(moved[n], ref[n]) for n in ref)
        model.params.load_data(snap)
        back = eng.params()
        for n in ref:
            assert np.array_equal(back[n], ref[n]), n
        host = {n: (0.5 * v).astype(np.float32) for n, v in ref.items()}
        model.params.load_data(host)
        got = eng.params()
        for n in ref:
            assert np.array_equal(got[n], host[n]), n
        snap.release()
    finally:
        ModelParams.copy_data, ModelParams.load_data = saved[0], saved[1]
        ModelParams._cmt_patched = False
        TR.DEFAULTS.clear()
        TR.DEFAULTS.update(saved[2])


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_pipeline_matches_sequential_steps(mode):
    """Engine.pipeline (batch i+1 staged on the host while step i runs, staging
    double-buffered, shapes changing between batches) gives exactly the losses,
    parameters and generator state of one Engine.step per batch."""
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    from tests.gpu_helpers import cfg_of
    d = O.Dims(96, 32, 256, 2, 0.2)
    params = scaled_params(d, 4, 0.1)
    shapes = [(7, 6, 8), (9, 5, 8), (7, 6, 8), (5, 8, 12)]
    batches = []
    for i, (S, T, B) in enumerate(shapes):
        src, sm, tgt, tm = O.synthetic_batch(96, S, T, B, seed=10 + i, ragged=True)
        batches.append(Batch(src, tgt, sm, tm))
    out = []
    for piped in (False, True):
        eng = Engine(cfg_of(d), mode=mode)
        eng.upload(params)
        gen = np.random.Generator(np.random.PCG64(9))
        if piped:
            losses = [l for l, _ in eng.pipeline(iter(batches), 1.0, 5.0, 0.1, gen)]
        else:
            losses = [eng.step(b, 1.0, 5.0, 0.1, gen)[0] for b in batches]
        out.append((losses, eng.params(), gen.bit_generator.state))
        eng.close()
    assert out[0][0] == out[1][0]
    assert out[0][2] == out[1][2]
    for n in out[0][1]:
        assert np.array_equal(out[0][1][n], out[1][1][n]), n


@pytest.mark.parametrize("tanh_", [True, False])
def test_ce_variants_agree(tanh_):
    """The two CE implementations (ce2=2 two-pass default, ce2=0 per-row
    kernel + separate column sums) give the same loss
    and gradients (including the output bias, a column sum of the CE
    gradient) within bf16 tolerance of the oracle, with and without the
    output tanh (training.py:96-120, layers.py:64-73)."""
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    from tests.gpu_helpers import cfg_of
    d = O.Dims(520, 64, 128, 1, 0.0, tanh_, False)
    params = scaled_params(d, 8, 0.3)
    src, sm, tgt, tm = O.synthetic_batch(520, 7, 9, 20, seed=3, ragged=True)
    ol, _, og, _, _ = oracle_step(d, params, (src, sm, tgt, tm), 0.1, 1.0, 5.0, 1, update=False)
    for ce2 in (2, 0):
        eng = Engine(cfg_of(d), mode="bf16")
        eng.set_option("ce2", ce2)
        eng.upload(params)
        loss, _ = eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, None, update=False)
        grads = eng.grads()
        eng.close()
        assert abs(loss - ol) <= BF16_TOL * abs(ol), ce2
        for n in ("out.w", "out.b", "att.w_c.w", "tgt_embed"):
            assert O.norm_rel_err(grads[n], og[n]) < BF16_TOL, (ce2, n)


def test_pipeline_numeric_error_surfaces_at_collection():
    """Engine.pipeline: a non-finite step raises NumericError when its result is
    collected, before the next batch is launched, and the device skipped its
    update (training.py:128-135, 148-155)."""
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.errors import NumericError
    from paper_1802_07170_b200.model import Batch
    from tests.gpu_helpers import cfg_of
    d, params, (src, sm, tgt, tm) = _small()
    params = {k: v.copy() for k, v in params.items()}
    params["out.w"][5, 3] = np.nan
    eng = Engine(cfg_of(d), mode="bf16")
    eng.upload(params)
    gen = eng.pipeline(iter([Batch(src, tgt, sm, tm)] * 3), 1.0, 5.0, 0.1, np.random.default_rng(0))
    with pytest.raises(NumericError):
        next(gen)
    after = eng.params()
    for n in params:
        assert np.array_equal(after[n], params[n], equal_nan=True), n
    eng.close()
