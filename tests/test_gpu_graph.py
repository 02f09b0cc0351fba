"""Captured-graph steps equal eager steps bit for bit.

The engine captures a step into a CUDA graph the second time a batch shape is
run and replays it afterwards; every per-batch value (generator state, lr,
clip, smoothing, 1/ntok, unique embedding rows, ids, masks, segments) is read
from device memory.  These tests run the same sequence of batches through an
engine with graphs off and one with graphs on (captured on a shape's first
run) and require identical losses, norms, generator advances and weights:
batches of one shape with different ids, ragged masks and unique-row counts,
interleaved shapes, INFER passes (dev_entropy, training.py:162-182), a
learnable change (training.py:128-139) and a non-finite step (weights kept).
"""

import numpy as np
import pytest

from oracle import minmt_oracle as O
from tests.gpu_helpers import cfg_of, scaled_params

pytestmark = pytest.mark.gpu


def _engine(d, params, mode, graph):
    from paper_1802_07170_b200.engine import Engine
    eng = Engine(cfg_of(d), mode=mode)
    eng.set_option("graph", graph)
    eng.upload(params)
    return eng


def _batches(V, shapes, seed):
    out = []
    for i, (S, T, B) in enumerate(shapes):
        out.append(O.synthetic_batch(V, S, T, B, seed=seed + i, ragged=(i % 2 == 1)))
    return out


def _run(eng, batches, seed, lrs, infer_every=0):
    from paper_1802_07170_b200.model import Batch
    gen = np.random.Generator(np.random.PCG64(seed))
    res = []
    for i, (src, sm, tgt, tm) in enumerate(batches):
        loss, norm = eng.step(Batch(src, tgt, sm, tm), lrs[i % len(lrs)], 1.0 + 0.5 * i, 0.1, gen)
        res.append((loss, norm))
        if infer_every and i % infer_every == 0:
            eng.stage(src, sm, tgt, tm)
            r = eng.run(0.0, None, 0.0, None, update=False, infer=True)
            res.append((r.loss_sum, r.ntok))
    return res, gen.bit_generator.state["state"]["state"], eng.params()


@pytest.mark.parametrize("mode", ["bf16", "fp32"])
def test_graph_steps_equal_eager(mode):
    V = 304
    d = O.Dims(V, 128, 256, 2, 0.2)
    params = scaled_params(d, 11, 0.1)
    shapes = [(9, 7, 16)] * 4 + [(6, 10, 16), (9, 7, 16), (6, 10, 16), (9, 7, 16)]
    batches = _batches(V, shapes, 100)
    out = {}
    for graph in (0, 2):
        eng = _engine(d, params, mode, graph)
        out[graph] = _run(eng, batches, 7, [1.0, 0.5], infer_every=3)
        replays, n_graphs = eng.stat("graph_replays")
        eng.close()
        if graph:
            assert replays >= len(batches) and n_graphs >= 3  # two train shapes + INFER
        else:
            assert replays == 0
    (r0, s0, p0), (r1, s1, p1) = out[0], out[2]
    assert r0 == r1
    assert s0 == s1
    for k in p0:
        assert np.array_equal(p0[k], p1[k]), k


def test_graph_recaptures_after_learnable_change():
    V = 304
    d = O.Dims(V, 128, 256, 1, 0.0)
    params = scaled_params(d, 12, 0.1)
    batches = _batches(V, [(8, 8, 16)] * 3, 200)
    out = {}
    for graph in (0, 1):
        from paper_1802_07170_b200.model import Batch
        eng = _engine(d, params, "bf16", graph)
        gen = np.random.Generator(np.random.PCG64(3))
        losses = []
        for i, (src, sm, tgt, tm) in enumerate(batches * 2):
            if i == 3:
                eng.set_learnable({"out.w": False, "src_embed": False})
            losses.append(eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, gen))
        out[graph] = (losses, eng.params())
        eng.close()
    assert out[0][0] == out[1][0]
    for k in out[0][1]:
        assert np.array_equal(out[0][1][k], out[1][1][k]), k


def test_graph_nonfinite_step_keeps_weights():
    from paper_1802_07170_b200.errors import NumericError
    from paper_1802_07170_b200.model import Batch
    V = 304
    d = O.Dims(V, 128, 256, 1, 0.0)
    params = scaled_params(d, 13, 0.1)
    (src, sm, tgt, tm), = _batches(V, [(8, 8, 16)], 300)
    eng = _engine(d, params, "bf16", 2)
    eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, None)  # captured, then replayed below
    bad = eng.params()
    bad["out.w"][3, 5] = np.nan  # non-finite logits (training.py:96-120 raises NumericError)
    eng.upload(bad)
    with pytest.raises(NumericError):
        eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, None)
    replays, _ = eng.stat("graph_replays")
    after = eng.params()
    eng.close()
    assert replays == 2
    for k in bad:
        assert np.array_equal(bad[k], after[k], equal_nan=True), k


def test_graph_probes_record_every_replay():
    """bench.py's kernel-class probes (CUDA events around the logits GEMM and the
    recurrent scans) stay inside the captured step: each replay records fresh
    events into the graph's record nodes."""
    from paper_1802_07170_b200.model import Batch
    V = 304
    d = O.Dims(V, 128, 256, 2, 0.2)
    params = scaled_params(d, 14, 0.1)
    (src, sm, tgt, tm), = _batches(V, [(8, 8, 16)], 400)
    counts = {}
    for graph in (0, 2):
        eng = _engine(d, params, "bf16", graph)
        eng.set_option("time_dominant", 7)
        gen = np.random.Generator(np.random.PCG64(1))
        for _ in range(5):
            eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, gen)
        counts[graph] = [eng.stat(f"probe_ms:{c}") for c in (0, 1, 2)]
        for _ in range(3):
            eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, gen)
        again = [eng.stat(f"probe_ms:{c}") for c in (0, 1, 2)]
        eng.close()
        for (ms, n), (ms2, n2) in zip(counts[graph], again):
            assert n > 0 and ms > 0 and n2 * 5 == n * 3 and ms2 > 0
    assert [n for _, n in counts[0]] == [n for _, n in counts[2]]


@pytest.mark.parametrize("shared", [False, True])
def test_device_segments_equal_host_segments(shared):
    """Embedding segments built in the step (segments_kernel: stable radix sort
    of the positions by id, unique ids, offsets) give the same embedding grads
    and updates as the host staging sort (np.add.at order, tensor.py:191-205)."""
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    V = 304
    d = O.Dims(V, 128, 256, 1, 0.0, shared_embeddings=shared)
    params = scaled_params(d, 15, 0.1)
    batches = _batches(V, [(9, 7, 16), (9, 7, 16), (5, 12, 24)], 500)
    res = {}
    for seg_dev in (0, 1):
        eng = Engine(cfg_of(d), mode="bf16")
        eng.set_option("seg_dev", seg_dev)
        eng.upload(params)
        gen = np.random.Generator(np.random.PCG64(2))
        out = []
        for src, sm, tgt, tm in batches:
            out.append(eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, gen))
        src, sm, tgt, tm = batches[0]
        eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, gen, update=False)
        rows = [eng.staged_rows(t) for t in range(eng.n_tables)]
        res[seg_dev] = (out, eng.grads(), eng.params(), rows)
        eng.close()
    assert res[0][0] == res[1][0]
    for k in res[0][1]:
        assert np.array_equal(res[0][1][k], res[1][1][k]), k
        assert np.array_equal(res[0][2][k], res[1][2][k]), k
    for a, b in zip(res[0][3], res[1][3]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("L", [1, 3])
def test_masks_ahead_equal_fused_dropout(L):
    """Dropout masks generated beside the recurrent scans (dropout_mask_kernel on
    the idle SMs) and applied at the sites (dropout_apply_kernel) equal the fused
    draw-and-apply kernel bit for bit: losses, generator advance, weights."""
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    V = 304
    d = O.Dims(V, 128, 256, L, 0.3)
    params = scaled_params(d, 16, 0.1)
    batches = _batches(V, [(9, 7, 16), (9, 7, 16), (9, 7, 16)], 600)
    res = {}
    for ahead in (0, 1):
        eng = Engine(cfg_of(d), mode="bf16")
        eng.set_option("mask_ahead", ahead)
        eng.upload(params)
        gen = np.random.Generator(np.random.PCG64(4))
        out = [eng.step(Batch(src, tgt, sm, tm), 1.0, 5.0, 0.1, gen) for src, sm, tgt, tm in batches]
        res[ahead] = (out, gen.bit_generator.state["state"]["state"], eng.params())
        eng.close()
    assert res[0][0] == res[1][0] and res[0][1] == res[1][1]
    for k in res[0][2]:
        assert np.array_equal(res[0][2][k], res[1][2][k]), k
