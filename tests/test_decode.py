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


def _setup(name, mode="fp32"):
    from paper_1802_07170_b200 import decoding as D
    from paper_1802_07170_b200.engine import Engine
    g = load()
    p = f"{name}/"
    model = model_of(g, name)
    eng = Engine(model.config, mode=mode)
    eng.upload(model.params)
    cfg = D.DecodeConfig(beam_size=int(g[p + "beam"]), length_penalty_alpha=float(g[p + "alpha"]),
                         n_best=int(g[p + "n_best"]))
    srcs = [[int(x) for x in g[f"{p}s{i}/src"]] for i in range(int(g[p + "n_sent"]))]
    return D, g, p, model, eng, cfg, srcs


def _close(a, b):
    return abs(a - b) <= 1e-4 * max(1.0, abs(b))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["d_deep", "d_shared", "d_wide"])
def test_decode_fp32_matches_reference(name):
    """fp32 validation mode, device beam search one sentence at a time: greedy
    and beam outputs (tokens, truncation, n-best lists) identical to the
    reference's, scores and log-probs within 1e-4 relative."""
    D, g, p, model, eng, cfg, srcs = _setup(name)
    for i, src in enumerate(srcs):
        q = f"{p}s{i}/"
        gr = D.greedy_decode(src, model, int(g[p + "greedy_len"]), engine=eng)
        assert gr.tokens == [int(x) for x in g[q + "greedy_tokens"]], (name, i)
        assert gr.truncated == bool(g[q + "greedy_truncated"])
        assert _close(gr.log_prob, float(g[q + "greedy_logprob"])) and gr.score == gr.log_prob
        t = D.beam_search(src, model, cfg, engine=eng)
        assert t.tokens == [int(x) for x in g[q + "beam_tokens"]], (name, i)
        assert t.truncated == bool(g[q + "beam_truncated"]), (name, i)
        assert _close(t.score, float(g[q + "beam_score"])) and _close(t.log_prob, float(g[q + "beam_logprob"]))
        assert len(t.n_best) == int(g[q + "nbest_n"])
        for j, (tk, sc, _) in enumerate(t.n_best):
            assert tk == [int(x) for x in g[q + f"nbest{j}_tokens"]], (name, i, j)
            assert _close(sc, float(g[q + f"nbest{j}_score"]))
    eng.close()


def _bf16_model():
    from paper_1802_07170_b200.model import Model, ModelConfig, Rng
    cfg = ModelConfig(304, 64, 256, 2, 0.2, True, False)  # bf16 needs multiples of 8
    model = Model.new(cfg, Rng(31))
    ir = Rng(1031)
    for b in model.params.blocks():
        b.var.data[:] = ir.uniform(-0.15, 0.15, b.var.shape, dtype=np.float32)
    return model


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_batched_search_equals_one_sentence_at_a_time(mode):
    """All sentences (different lengths: a padded, masked batch) in one device
    search give exactly the per-sentence results: the padded encoder carries
    state through padding and masks it out of attention exactly, and every
    row of a decoder step is independent of the others."""
    D, g, p, model, eng, cfg, srcs = _setup("d_wide", "fp32")
    if mode == "bf16":
        from paper_1802_07170_b200.engine import Engine
        eng.close()
        model = _bf16_model()
        eng = Engine(model.config, mode="bf16")
        eng.upload(model.params)
        r = np.random.default_rng(7)
        srcs = [list(r.integers(4, 304, n)) for n in (3, 9, 1, 14, 6, 6, 11)]
    cfg.n_best = 3
    caps = [D.length_cap(cfg, len(s)) for s in srcs]
    together = D._run(eng, srcs, cfg.beam_size, cfg.n_best, caps, cfg.length_penalty_alpha)
    for src, cap, t in zip(srcs, caps, together):
        (one,) = D._run(eng, [src], cfg.beam_size, cfg.n_best, [cap], cfg.length_penalty_alpha)
        assert one == t
    eng.close()


@pytest.mark.gpu
def test_translate_batch_order_and_records():
    """translate_batch (decoding.py:174-205): input order kept, empty lines
    empty, n-best records '<i> ||| tokens ||| score' equal to per-line beam
    search; bad ids raise ConfigError naming the line."""
    from paper_1802_07170_b200.errors import ConfigError
    D, g, p, model, eng, cfg, srcs = _setup("d_shared")

    class Vocab:
        def encode(self, words):
            return [int(w) for w in words]

        def decode(self, ids):
            return [str(x) for x in ids]
    cfg.n_best = 2
    lines = [" ".join(map(str, s)) for s in srcs]
    lines.insert(2, "   ")
    outputs, records = D.translate_batch(lines, model, Vocab(), cfg, engine=eng, batch_sentences=3)
    assert outputs[2] == ""
    expect = []
    for i, line in enumerate(lines):
        if not line.split():
            continue
        t = D.beam_search([int(w) for w in line.split()], model, cfg, engine=eng)
        assert outputs[i] == " ".join(map(str, t.tokens))
        expect += [f"{i} ||| {' '.join(map(str, tk))} ||| {sc:.6f}" for tk, sc, _ in t.n_best[:2]]
    assert records == expect
    with pytest.raises(ConfigError, match="line 2"):
        D.translate_batch(["4 5", f"6 {model.config.vocab_size}"], model, Vocab(), cfg, engine=eng)
    with pytest.raises(ConfigError):
        D.beam_search([], model, cfg, engine=eng)
    eng.close()


@pytest.mark.gpu
def test_decode_bf16_close_to_fp32():
    """bf16 production mode against the fp32 validation mode (pinned to the
    reference above): where greedy decoding picks the same tokens, the
    sequence log-probs agree within 2e-2 relative."""
    from paper_1802_07170_b200 import decoding as D
    from paper_1802_07170_b200.engine import Engine
    model = _bf16_model()
    cfg = model.config
    engs = {m: Engine(cfg, mode=m) for m in ("fp32", "bf16")}
    for e in engs.values():
        e.upload(model.params)
    same = 0
    srcs = ([14, 209, 129], [193, 82, 42, 183, 37, 6, 9, 11], [35], [7, 8, 9, 10, 11, 12])
    for src in srcs:
        a = D.greedy_decode(src, model, 6, engine=engs["fp32"])
        b = D.greedy_decode(src, model, 6, engine=engs["bf16"])
        if a.tokens == b.tokens:
            same += 1
            assert abs(a.log_prob - b.log_prob) <= 2e-2 * abs(a.log_prob), (src, a, b)
    assert same >= len(srcs) // 2
    for e in engs.values():
        e.close()
