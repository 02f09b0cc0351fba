"""Generate golden fixtures by running the REAL reference (minmt) train step.

Run in the authoring container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``minmt`` from /root/reference/pkg/src (read-only), runs
``minmt.training.train_step`` (training.py:145-159) on seeded inputs and
records loss, every per-block gradient (captured by wrapping
``minmt.training.sgd_step`` before it zeroes them, training.py:140-141), the
updated weights, the gradient norm and the dropout RNG state after the step.

Small cases store full arrays; the ``tiny`` case (BASELINE.json configs[0])
stores per-block checksums only, to keep the fixture small.  The GPU box never
reads /root/reference: tests load these .npz files instead.
"""

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import minmt.training as mt  # noqa: E402
from minmt.data import Batch  # noqa: E402
from minmt.model import Model, ModelConfig  # noqa: E402
from minmt.tensor import Rng  # noqa: E402

from oracle.minmt_oracle import synthetic_batch  # noqa: E402

CASES = {
    # reference toy fixture (pkg/tests/test_model.py:26-47), weights re-drawn at +-0.8
    "toy": dict(V=11, E=4, H=4, L=2, dropout=0.0, tanh=True, shared=False,
                src=[[4, 5], [6, 7], [8, 0]], src_mask=[[1, 1], [1, 1], [1, 0]],
                tgt=[[5, 6], [7, 8], [3, 3]], tgt_mask=[[1, 1], [1, 1], [1, 1]],
                scale=0.8, seed=0, eps=0.1, lr=1.0, clip=5.0),
    "toy_dropout": dict(V=11, E=4, H=4, L=2, dropout=0.25, tanh=True, shared=False,
                        src=[[4, 5], [6, 7], [8, 0]], src_mask=[[1, 1], [1, 1], [1, 0]],
                        tgt=[[5, 6], [7, 8], [3, 3]], tgt_mask=[[1, 1], [1, 1], [1, 1]],
                        scale=0.8, seed=3, eps=0.1, lr=0.5, clip=5.0),
    "ragged_clip": dict(V=37, E=8, H=16, L=3, dropout=0.3, tanh=True, shared=False,
                        S=7, T=6, B=5, ragged=True, scale=0.5, seed=7, eps=0.1, lr=1.0, clip=0.05),
    "notanh_shared": dict(V=29, E=8, H=8, L=2, dropout=0.0, tanh=False, shared=True,
                          S=5, T=4, B=4, ragged=True, scale=0.6, seed=11, eps=0.2, lr=0.7, clip=None),
    "deep_noclip": dict(V=41, E=16, H=8, L=4, dropout=0.1, tanh=True, shared=False,
                        S=4, T=5, B=8, ragged=False, scale=0.3, seed=13, eps=0.0, lr=2.0, clip=None),
    # BASELINE.json configs[0]: Model.new init (+-0.1, forget bias 1), checksums only
    "tiny": dict(V=1000, E=128, H=128, L=1, dropout=0.2, tanh=True, shared=False,
                 S=20, T=20, B=16, ragged=True, scale=None, seed=1, eps=0.1, lr=1.0, clip=5.0,
                 checksums=True),
}

SAMPLE = 16


def checksum(a):
    a = np.asarray(a, np.float64).ravel()
    idx = np.linspace(0, a.size - 1, num=min(SAMPLE, a.size)).astype(np.int64)
    return np.concatenate([[a.sum(), (a * a).sum(), np.abs(a).sum(), a.size], a[idx]])


def run(name, c):
    cfg = ModelConfig(vocab_size=c["V"], embedding_size=c["E"], hidden_size=c["H"], depth=c["L"],
                      dropout=c["dropout"], output_tanh=c["tanh"], shared_embeddings=c["shared"])
    model = Model.new(cfg, Rng(c["seed"]))
    if c["scale"] is not None:
        ir = Rng(c["seed"] + 1000)
        for b in model.params.blocks():
            b.var.data[:] = ir.uniform(-c["scale"], c["scale"], b.var.shape, dtype=np.float32)
    if "src" in c:
        src = np.array(c["src"], np.int64)
        sm = np.array(c["src_mask"], np.float32)
        tgt = np.array(c["tgt"], np.int64)
        tm = np.array(c["tgt_mask"], np.float32)
    else:
        src, sm, tgt, tm = synthetic_batch(c["V"], c["S"], c["T"], c["B"], seed=c["seed"],
                                           ragged=c["ragged"])
    batch = Batch(src, tgt, sm, tm, [], [], [])
    init = {b.name: b.var.data.copy() for b in model.params.blocks()}
    captured = {}
    real_sgd = mt.sgd_step

    def spy(blocks, lr, clip_norm=None):
        for b in blocks:
            captured[b.name] = b.var.grad.copy()
        n = real_sgd(blocks, lr, clip_norm)
        captured["__norm__"] = n
        return n

    mt.sgd_step = spy
    rng = Rng(c["seed"] + 5)
    try:
        tcfg = mt.TrainConfig(label_smoothing=c["eps"], grad_clip_norm=c["clip"])
        loss = mt.train_step(model, batch, tcfg, c["lr"], rng)
    finally:
        mt.sgd_step = real_sgd
    state = rng.gen.bit_generator.state["state"]
    out = dict(
        V=c["V"], E=c["E"], H=c["H"], L=c["L"], dropout=c["dropout"], tanh=int(c["tanh"]),
        shared=int(c["shared"]), seed=c["seed"], eps=c["eps"], lr=c["lr"],
        clip=(-1.0 if c["clip"] is None else c["clip"]), scale=(-1.0 if c["scale"] is None else c["scale"]),
        src=src, src_mask=sm, tgt=tgt, tgt_mask=tm, loss=loss, norm=captured["__norm__"],
        rng_state=np.array([state["state"] >> 64, state["state"] & ((1 << 64) - 1),
                            state["inc"] >> 64, state["inc"] & ((1 << 64) - 1)], dtype=np.uint64),
        names=np.array([b.name for b in model.params.blocks()]),
    )
    for b in model.params.blocks():
        if c.get("checksums"):
            out[f"init:{b.name}"] = checksum(init[b.name])
            out[f"grad:{b.name}"] = checksum(captured[b.name])
            out[f"new:{b.name}"] = checksum(b.var.data)
        else:
            out[f"init:{b.name}"] = init[b.name]
            out[f"grad:{b.name}"] = captured[b.name]
            out[f"new:{b.name}"] = b.var.data.copy()
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: loss={loss:.8f} norm={captured['__norm__']:.6f} -> {path} ({os.path.getsize(path)} B)")


if __name__ == "__main__":
    for n, c in CASES.items():
        run(n, c)
