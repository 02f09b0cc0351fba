"""Rebuild the models of tests/golden/decode.npz (make_decode_golden.py) with
this package's Model/Rng mirrors: Model.new(cfg, Rng(seed)), every block
redrawn from Rng(seed + 1000).uniform(+-scale), EOS bias raised."""

import os

import numpy as np

from paper_1802_07170_b200.model import Model, ModelConfig, Rng

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "decode.npz")


def load():
    return np.load(PATH, allow_pickle=False)


def model_of(g, name):
    p = f"{name}/"
    cfg = ModelConfig(int(g[p + "V"]), int(g[p + "E"]), int(g[p + "H"]), int(g[p + "L"]), 0.2,
                      bool(g[p + "tanh"]), bool(g[p + "shared"]))
    seed = int(g[p + "seed"])
    model = Model.new(cfg, Rng(seed))
    ir = Rng(seed + 1000)
    scale = float(g[p + "scale"])
    for b in model.params.blocks():
        b.var.data[:] = ir.uniform(-scale, scale, b.var.shape, dtype=np.float32)
    ob = next(b for b in model.params.blocks() if b.name == "out.b")
    ob.var.data[3, 0] += np.float32(float(g[p + "eos_bias"]))
    return model
