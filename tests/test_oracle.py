"""Pin the CPU oracle to the reference: golden fixtures + the reference's own KATs.

Fixtures come from tests/golden/make_golden.py (the real minmt train_step).
Tolerances: fp32 restatement vs fp32 reference differ only in summation order.
"""

import math

import numpy as np
import pytest

from oracle import minmt_oracle as O
from paper_1802_07170_b200.model import Model, ModelConfig, Rng

SMALL = ["toy", "toy_dropout", "ragged_clip", "notanh_shared", "deep_noclip"]


def dims_of(g):
    return O.Dims(int(g["V"]), int(g["E"]), int(g["H"]), int(g["L"]), float(g["dropout"]),
                  bool(g["tanh"]), bool(g["shared"]))


def run_oracle(g, params):
    d = dims_of(g)
    gen = np.random.Generator(np.random.PCG64(int(g["seed"]) + 5))
    clip = None if float(g["clip"]) < 0 else float(g["clip"])
    batch = (g["src"], g["src_mask"], g["tgt"], g["tgt_mask"])
    loss, norm, grads = O.train_step(params, d, batch, float(g["eps"]), float(g["lr"]), clip, gen)
    return loss, norm, grads, gen


@pytest.mark.parametrize("case", SMALL)
def test_oracle_matches_reference_golden(golden, case):
    g = golden(case)
    names = [str(n) for n in g["names"]]
    assert names == [n for n, _ in O.registry(dims_of(g))]
    params = {n: g[f"init:{n}"].copy() for n in names}
    loss, norm, grads, gen = run_oracle(g, params)
    assert abs(loss - float(g["loss"])) <= 1e-6 * abs(float(g["loss"]))
    assert abs(norm - float(g["norm"])) <= 1e-5 * float(g["norm"])
    for n in names:
        assert O.norm_rel_err(grads[n], g[f"grad:{n}"]) < 1e-5, n
        assert O.norm_rel_err(params[n], g[f"new:{n}"]) < 1e-6, n
    # the oracle consumed exactly the reference's dropout draws
    st = gen.bit_generator.state["state"]
    ref = [int(x) for x in g["rng_state"]]
    assert (st["state"] >> 64, st["state"] & ((1 << 64) - 1)) == (ref[0], ref[1])


def test_oracle_tiny_checksums_and_mirror_init(golden):
    """BASELINE configs[0]; also pins the host mirror's Model.new draw order."""
    g = golden("tiny")
    cfg = ModelConfig(int(g["V"]), int(g["E"]), int(g["H"]), int(g["L"]), float(g["dropout"]))
    model = Model.new(cfg, Rng(int(g["seed"])))
    params = {}
    for b in model.params.blocks():
        ck = g[f"init:{b.name}"]
        mine = np.asarray(b.var.data, np.float64).ravel()
        assert mine.sum() == ck[0] and (mine * mine).sum() == ck[1], b.name  # bit-exact init
        params[b.name] = b.var.data.copy()
    loss, norm, grads, _ = run_oracle(g, params)
    assert abs(loss - float(g["loss"])) <= 1e-6 * float(g["loss"])
    assert abs(norm - float(g["norm"])) <= 1e-5 * float(g["norm"])
    for n in params:
        ck = g[f"grad:{n}"]
        gg = np.asarray(grads[n], np.float64).ravel()
        assert abs(math.sqrt((gg * gg).sum()) - math.sqrt(ck[1])) <= 1e-4 * math.sqrt(ck[1]) + 1e-12, n
        idx = np.linspace(0, gg.size - 1, num=min(16, gg.size)).astype(np.int64)
        scale = max(np.abs(gg).max(), 1e-30)
        assert np.abs(gg[idx] - ck[4:4 + idx.size]).max() <= 1e-4 * scale, n


# ---- known-answer tests the reference's own suite holds ----

def test_kat_label_smoothing_value():
    # pkg/tests/test_training.py:43-47: eps=0.1, V=4, p=[.7,.1,.1,.1] -> 0.5027
    p = np.array([[0.7], [0.1], [0.1], [0.1]])
    loss, _ = O.smoothed_loss(np.log(p), np.array([0]), 0.1, None)
    assert abs(loss - 0.5027) < 1e-4


def test_kat_uniform_prediction_is_log_v():
    # pkg/tests/test_training.py:36-41
    V = 7
    lp = np.full((V, 3), -math.log(V))
    for eps in (0.0, 0.1, 0.5, 0.9):
        loss, _ = O.smoothed_loss(lp, np.array([1, 2, 3]), eps, None)
        assert abs(loss - math.log(V)) < 1e-12


def test_kat_softmax_values():
    # pkg/tests/test_tensor.py:71-74
    p = O.softmax_cols(np.array([[1.0], [2.0], [3.0]]))
    assert np.allclose(p[:, 0], [0.09003057, 0.24472847, 0.66524096], atol=1e-8)


def test_kat_masked_positions_zero_grad():
    # pkg/tests/test_training.py:61-64
    lp = O.log_softmax_cols(np.random.default_rng(0).normal(size=(4, 3)))
    _, d = O.smoothed_loss(lp, np.array([0, 1, 2]), 0.1, np.array([1.0, 0.0, 1.0]))
    assert not d[:, 1].any()


def test_kat_masked_alignment_exact_zero():
    # pkg/tests/test_attention.py:61-71: masked source positions get alpha == 0.0
    d = O.Dims(11, 4, 4, 1, 0.0)
    p = O.init_params(d, np.random.default_rng(0))
    src = np.array([[4, 5], [6, 0], [7, 0]])
    sm = np.array([[1, 1], [1, 0], [1, 0]], np.float32)
    tgt = np.array([[5, 6], [3, 3]])
    _, _, aux = O.forward_backward(p, d, src, sm, tgt, np.ones((2, 2), np.float32), 0.1,
                                   want_grads=False)
    a = aux["alpha"].reshape(3, 2, 2)
    assert (a[1:, :, 1] == 0.0).all() and (a[:, :, 0] > 0).all()


def test_kat_padding_carries_state():
    # pkg/tests/test_layers.py:179-189: padded steps carry the previous state
    d = O.Dims(11, 4, 4, 1, 0.0)
    p = O.init_params(d, np.random.default_rng(1))
    x = np.random.default_rng(2).normal(size=(4, 3 * 2)).astype(np.float32)
    mask = np.array([[1, 1], [1, 0], [1, 0]], np.float32)
    y, (h, c), _ = O.lstm_scan(p, "enc.l1.fwd", x, 3, 2, mask=mask)
    y3 = y.reshape(4, 3, 2)
    assert np.array_equal(y3[:, 1, 1], y3[:, 0, 1]) and np.array_equal(h[:, 1], y3[:, 0, 1])


def test_errors_bad_id_and_fully_masked():
    d = O.Dims(11, 4, 4, 1, 0.0)
    p = O.init_params(d, np.random.default_rng(0))
    with pytest.raises(O.OracleError) as e:
        O.forward_backward(p, d, np.array([[11]]), np.ones((1, 1)), np.array([[3]]), np.ones((1, 1)), 0.1)
    assert e.value.kind == "ConfigError"
    with pytest.raises(O.OracleError) as e:
        O.forward_backward(p, d, np.array([[4, 5]]), np.array([[1, 0]]), np.array([[3, 3]]),
                           np.ones((1, 2)), 0.1)
    assert e.value.kind == "MaskError"


def test_sgd_nonfinite_aborts_without_update():
    # pkg/tests/test_training.py:116-121
    p = {"w": np.ones((1, 1), np.float32)}
    g = {"w": np.full((1, 1), np.nan, np.float32)}
    with pytest.raises(O.OracleError):
        O.sgd_step(p, g, ["w"], 1.0, None)
    assert p["w"][0, 0] == 1.0


@pytest.mark.parametrize("case", SMALL)
def test_oracle_dev_entropy_matches_reference(golden, case):
    """dev_entropy (training.py:162-182) against values produced by the real
    reference (tests/golden/make_dev_golden.py)."""
    g = golden(case)
    dv = golden("dev_entropy")
    names = [str(n) for n in g["names"]]
    params = {n: g[f"init:{n}"].copy() for n in names}
    batches = [(g["src"], g["src_mask"], g["tgt"], g["tgt_mask"]),
               (dv[f"{case}:src2"], dv[f"{case}:sm2"], dv[f"{case}:tgt2"], dv[f"{case}:tm2"])]
    val = O.dev_entropy(params, dims_of(g), batches)
    assert abs(val - float(dv[f"{case}:value"])) <= 1e-6 * abs(float(dv[f"{case}:value"]))
