"""Golden values of the reference's dev_entropy (training.py:162-182).

Run in the authoring container (needs /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_dev_golden.py

For each small train-step fixture it rebuilds the reference Model with the
fixture's initial weights and evaluates ``minmt.training.dev_entropy`` on two
batches: the fixture batch and a second seeded (ragged) batch.  Stores the
batches and the value in tests/golden/dev_entropy.npz.
"""

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import minmt.training as mt  # noqa: E402
from minmt.data import Batch  # noqa: E402
from minmt.model import Model, ModelConfig  # noqa: E402
from minmt.tensor import Rng  # noqa: E402

from oracle.minmt_oracle import synthetic_batch  # noqa: E402

CASES = ["toy", "toy_dropout", "ragged_clip", "notanh_shared", "deep_noclip"]

if __name__ == "__main__":
    out = {}
    for name in CASES:
        g = np.load(os.path.join(HERE, f"{name}.npz"))
        cfg = ModelConfig(vocab_size=int(g["V"]), embedding_size=int(g["E"]), hidden_size=int(g["H"]),
                          depth=int(g["L"]), dropout=float(g["dropout"]), output_tanh=bool(g["tanh"]),
                          shared_embeddings=bool(g["shared"]))
        model = Model.new(cfg, Rng(0))
        for b in model.params.blocks():
            b.var.data[:] = g[f"init:{b.name}"]
        S, B = g["src"].shape
        T = g["tgt"].shape[0]
        src2, sm2, tgt2, tm2 = synthetic_batch(int(g["V"]), S + 1, T + 2, B, seed=int(g["seed"]) + 77, ragged=True)
        batches = [Batch(g["src"], g["tgt"], g["src_mask"], g["tgt_mask"], [], [], []),
                   Batch(src2, tgt2, sm2, tm2, [], [], [])]
        val = mt.dev_entropy(model, batches)
        out[f"{name}:value"] = np.float64(val)
        for k, a in (("src2", src2), ("sm2", sm2), ("tgt2", tgt2), ("tm2", tm2)):
            out[f"{name}:{k}"] = a
        print(f"{name}: dev_entropy = {val:.10f}")
    path = os.path.join(HERE, "dev_entropy.npz")
    np.savez_compressed(path, **out)
    print("->", path, os.path.getsize(path), "B")
