"""GPU translation against the reference's own decoding
outputs (tests/golden/decode.npz, made by make_decode_golden.py from
minmt.decoding / minmt.model, decoding.py:89-187, model.py:180-236)."""

import numpy as np
import pytest

from tests.decode_fixture import load, model_of


def test_fixture_models_regenerate_exactly():
    """The decode fixtures store weight checksums; this package's Model.new and
    Rng rebuild those weights bit for bit (CPU)."""
    g = load()
    for name in g["cases"]:
        model = model_of(g, str(name))
        names = [str(n) for n in g[f"{name}/names"]]
        assert names == [b.name for b in model.params.blocks()]
        for b in model.params.blocks():
            a = b.var.data.astype(np.float64)
            ck = g[f"{name}/ck:{b.name}"]
            assert a.sum() == ck[0] and (a * a).sum() == ck[1], (name, b.name)


def _decoders(mode):
    from paper_1802_07170_b200 import decoding as D
    from paper_1802_07170_b200.engine import Engine
    return D, Engine


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["d_deep", "d_shared", "d_wide"])
def test_decode_fp32_matches_reference(name):
    """fp32 validation mode: first-step log-probs within 1e-4 (norm-relative),
    greedy and beam outputs (tokens, truncation, n-best) identical, scores and
    log-probs within 1e-4 relative."""
    D, Engine = _decoders("fp32")
    g = load()
    p = f"{name}/"
    model = model_of(g, name)
    eng = Engine(model.config, mode="fp32")
    eng.upload(model.params)
    cfg = D.DecodeConfig(beam_size=int(g[p + "beam"]), length_penalty_alpha=float(g[p + "alpha"]),
                         n_best=int(g[p + "n_best"]))
    for i in range(int(g[p + "n_sent"])):
        q = f"{p}s{i}/"
        src = [int(x) for x in g[q + "src"]]
        eng.decode_begin(src)
        V = model.config.vocab_size
        vals, toks = eng.decode_step([2], None, min(32, V))
        ref = g[q + "first_logprobs"]
        order = np.lexsort((np.arange(V), -ref))[: vals.shape[1]]
        assert np.max(np.abs(vals[0] - ref[toks[0]])) <= 1e-4 * np.max(np.abs(ref)), (name, i)
        assert list(toks[0]) == list(order), (name, i)
        gr = D.greedy_decode(src, model, int(g[p + "greedy_len"]), engine=eng)
        assert gr.tokens == [int(x) for x in g[q + "greedy_tokens"]], (name, i)
        assert gr.truncated == bool(g[q + "greedy_truncated"])
        assert abs(gr.log_prob - float(g[q + "greedy_logprob"])) <= 1e-4 * max(1.0, abs(gr.log_prob))
        t = D.beam_search(src, model, cfg, engine=eng)
        assert t.tokens == [int(x) for x in g[q + "beam_tokens"]], (name, i)
        assert t.truncated == bool(g[q + "beam_truncated"]), (name, i)
        assert abs(t.score - float(g[q + "beam_score"])) <= 1e-4 * max(1.0, abs(t.score))
        assert abs(t.log_prob - float(g[q + "beam_logprob"])) <= 1e-4 * max(1.0, abs(t.log_prob))
        assert len(t.n_best) == int(g[q + "nbest_n"])
        for j, (tk, sc, lpb) in enumerate(t.n_best):
            assert tk == [int(x) for x in g[q + f"nbest{j}_tokens"]], (name, i, j)
            assert abs(sc - float(g[q + f"nbest{j}_score"])) <= 1e-4 * max(1.0, abs(sc))
    eng.close()


@pytest.mark.gpu
def test_decode_bf16_matches_fp32():
    """bf16 production mode (bf16 weights, fp32 arithmetic) against the fp32
    validation mode, which the test above pins to the reference: the best
    tokens' log-probs of the first steps within 2e-2 norm-relative."""
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Model, ModelConfig, Rng
    cfg = ModelConfig(304, 64, 256, 2, 0.2, True, False)  # bf16 needs multiples of 8
    model = Model.new(cfg, Rng(31))
    ir = Rng(1031)
    for b in model.params.blocks():
        b.var.data[:] = ir.uniform(-0.15, 0.15, b.var.shape, dtype=np.float32)
    engs = {}
    for mode in ("fp32", "bf16"):
        engs[mode] = Engine(cfg, mode=mode)
        engs[mode].upload(model.params)
    for src in ([14, 209, 129], [193, 82, 42, 183, 37, 6, 9, 11], [35]):
        out = {}
        for mode, eng in engs.items():
            eng.decode_begin(src)
            v0, t0 = eng.decode_step([2], None, 8)
            v1, t1 = eng.decode_step([int(t0[0, 0]), int(t0[0, 1])], [0, 0], 8)
            out[mode] = (np.concatenate([v0[0], v1.ravel()]), np.concatenate([t0[0], t1.ravel()]))
        scale = np.max(np.abs(out["fp32"][0]))
        both = out["fp32"][1] == out["bf16"][1]  # compare where the same tokens were selected
        assert both.mean() > 0.5
        assert np.max(np.abs(out["fp32"][0][both] - out["bf16"][0][both])) <= 2e-2 * scale
    for eng in engs.values():
        eng.close()


@pytest.mark.gpu
def test_decode_errors_and_states():
    """Bad ids raise ConfigError; decode_step before decode_begin raises; a
    batched step over duplicated rows equals the single-row step (state
    gathering by parent index)."""
    from paper_1802_07170_b200.errors import ConfigError
    D, Engine = _decoders("fp32")
    g = load()
    model = model_of(g, "d_deep")
    eng = Engine(model.config, mode="fp32")
    eng.upload(model.params)
    with pytest.raises(ConfigError):
        eng.decode_step([2], None, 1)
    eng.decode_begin([5, 6, 7])
    v1, t1 = eng.decode_step([2], None, 4)
    v2, t2 = eng.decode_step([int(t1[0, 0]), int(t1[0, 1])], [0, 0], 4)
    eng.decode_begin([5, 6, 7])
    w1, _ = eng.decode_step([2, 2, 2], None, 4)
    assert np.array_equal(np.repeat(v1, 3, axis=0), w1)
    w2, u2 = eng.decode_step([int(t1[0, 1]), int(t1[0, 0])], [2, 1], 4)
    assert np.array_equal(w2[::-1], v2) and np.array_equal(u2[::-1], t2)
    with pytest.raises(ConfigError):
        eng.decode_step([model.config.vocab_size], [0], 1)
    with pytest.raises(ConfigError):
        eng.decode_begin([])
    eng.close()


@pytest.mark.gpu
def test_decode_wide_beam_rows_match_single_rows():
    """More than 16 live rows (two GEMV passes): every row equals the same row
    decoded alone."""
    from paper_1802_07170_b200.engine import Engine
    g = load()
    model = model_of(g, "d_wide")
    eng = Engine(model.config, mode="fp32")
    eng.upload(model.params)
    src = [int(x) for x in g["d_wide/s1/src"]]
    toks = [4 + 7 * i for i in range(20)]
    eng.decode_begin(src)
    eng.decode_step([2], None, 1)
    vw, tw = eng.decode_step(toks, [0] * 20, 5)
    for i in (0, 15, 16, 19):
        eng.decode_begin(src)
        eng.decode_step([2], None, 1)
        v1, t1 = eng.decode_step([toks[i]], [0], 5)
        assert np.array_equal(t1[0], tw[i]) and np.allclose(v1[0], vw[i], rtol=0, atol=1e-5), i
    eng.close()
