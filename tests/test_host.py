"""CPU-side checks: the C-ABI library loads and exports every declared symbol,
the host mirror matches the reference registry, and the PCG64 jump-ahead the
dropout kernel implements reproduces numpy's draws (algorithm check on CPU)."""

import os
import re

import numpy as np
import pytest

from oracle import minmt_oracle as O
from paper_1802_07170_b200 import _lib
from paper_1802_07170_b200.engine import dropout_draws, pcg_state
from paper_1802_07170_b200.model import Model, ModelConfig, Rng

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "cytonmt_b200.h")).read()
    return sorted(set(re.findall(r"\b(cmt_[a-z_]+)\s*\(", txt)))


def test_library_loads_and_exports_all_header_symbols():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 17
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == syms
    assert isinstance(lib.cmt_launch_count(), int)


def test_dp_status_combine_is_flagwise():
    """The ranks' status words are combined flag by flag (engine.cu data-parallel
    branch: spread, ncclMax, rebuild).  A SUM of the words would turn 4 ranks
    raising ST_LOGITS (2) into 8 = ST_NORM and 16 ranks raising it into 32,
    outside the abort mask; the flagwise rule keeps exactly the raised flags."""
    import ctypes
    lib = _lib.load()
    ST_SCORES, ST_LOGITS, ST_LOSS, ST_NORM = 1, 2, 4, 8

    def combine(words):
        arr = (ctypes.c_int * len(words))(*words)
        return lib.cmt_status_combine(arr, len(words))
    for n in (1, 2, 4, 8, 16):
        assert combine([ST_LOGITS] * n) == ST_LOGITS
        assert combine([0] * (n - 1) + [ST_NORM]) == ST_NORM
    assert combine([0, 0, 0]) == 0
    assert combine([ST_SCORES, ST_LOSS, 0, ST_SCORES | ST_NORM]) == ST_SCORES | ST_LOSS | ST_NORM
    assert sum([ST_LOGITS] * 4) == ST_NORM  # what the old SUM combine produced


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1802_07170_b200.engine import Engine
    with pytest.raises(Exception):
        Engine(ModelConfig(64, 16, 16, 1), mode="fp32")


@pytest.mark.parametrize("shared", [False, True])
def test_mirror_registry_matches_reference_order(shared):
    cfg = ModelConfig(50, 8, 16, 3, shared_embeddings=shared)
    m = Model.new(cfg, Rng(0))
    d = O.Dims(50, 8, 16, 3, shared_embeddings=shared)
    assert [(b.name, b.var.shape) for b in m.params.blocks()] == O.registry(d)


def test_dropout_draw_count_matches_oracle():
    cfg = ModelConfig(50, 8, 16, 3, dropout=0.3)
    d = O.Dims(50, 8, 16, 3, dropout=0.3)
    assert dropout_draws(cfg, 7, 5, 4) == O.dropout_draws(d, 7, 5, 4)


# ---- the device PCG64 algorithm, restated in Python (kernels.cuh pcg_advance/pcg_out) ----
MASK128 = (1 << 128) - 1
MULT = 0x2360ED051FC65DA44385DF649FCCF645


def py_advance(state, inc, delta):
    cm, cp, am, ap = MULT, inc, 1, 0
    while delta:
        if delta & 1:
            am = (am * cm) & MASK128
            ap = (ap * cm + cp) & MASK128
        cp = ((cm + 1) * cp) & MASK128
        cm = (cm * cm) & MASK128
        delta >>= 1
    return (am * state + ap) & MASK128


def py_out(s):
    x = ((s >> 64) ^ s) & ((1 << 64) - 1)
    rot = s >> 122
    return ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)


def test_pcg64_jump_ahead_reproduces_numpy_random():
    rng = Rng(5)
    sh, sl, ih, il = pcg_state(rng)
    state, inc = (sh << 64) | sl, (ih << 64) | il
    ref = rng.gen.random(size=5000)
    for i in [0, 1, 2, 17, 1000, 4999]:
        s = py_advance(state, inc, i + 1)
        assert (py_out(s) >> 11) * (1.0 / 9007199254740992.0) == ref[i]


def test_numpy_advance_matches_draw_count():
    a, b = Rng(9), Rng(9)
    a.gen.random(size=1234)
    b.gen.bit_generator.advance(1234)
    assert a.gen.bit_generator.state == b.gen.bit_generator.state
    assert a.gen.random() == b.gen.random()
