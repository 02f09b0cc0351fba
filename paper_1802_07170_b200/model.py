"""Host-side mirror of the reference's model / config / batch types.

The drop-in ``train_step`` accepts the reference's own objects (duck-typed:
``model.config`` fields and ``model.params.blocks()`` with ``.name`` and
``.var.data``/``.var.grad``).  This module provides identically shaped types so
the engine can be driven where the reference package is not installed (the GPU
box, the benchmark).  Semantics follow:

* ``Rng`` ............ pkg/src/minmt/tensor.py:39-62 (numpy PCG64 Generator)
* ``Variable`` ....... pkg/src/minmt/tensor.py:65-100
* ``ParamBlock`` ..... pkg/src/minmt/graph.py:20-31
* ``ModelConfig`` .... pkg/src/minmt/model.py:46-62
* ``ModelParams`` .... pkg/src/minmt/model.py:65-115 (registry order + init draw order)
* ``TrainConfig`` .... pkg/src/minmt/training.py:31-52
* ``Batch`` .......... pkg/src/minmt/data.py:108-122
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError, ShapeError

GATES = ("i", "f", "g", "o")
INIT_SCALE = 0.1
PAD, UNK, BOS, EOS = 0, 1, 2, 3


@dataclass
class Rng:
    """Seeded PCG64 stream; same seed, same draws as the reference's Rng."""

    seed: int
    algorithm: str = "pcg64"
    gen: np.random.Generator = field(init=False, repr=False)

    def __post_init__(self):
        self.gen = np.random.Generator(np.random.PCG64(self.seed))

    def uniform(self, low, high, shape, dtype=None):
        return self.gen.uniform(low, high, size=shape).astype(dtype or np.float32)

    def random(self, shape, dtype=None):
        return self.gen.random(size=shape).astype(dtype or np.float32)

    def permutation(self, n):
        return self.gen.permutation(n)

    def integers(self, low, high, shape=None):
        return self.gen.integers(low, high, size=shape)


class Variable:
    __slots__ = ("data", "grad")

    def __init__(self, data):
        data = np.asarray(data)
        if data.ndim != 2:
            raise ShapeError(f"Variable requires a 2-d matrix, got shape {data.shape}")
        self.data = data
        self.grad = np.zeros_like(data)

    @property
    def shape(self):
        return self.data.shape

    @property
    def dtype(self):
        return self.data.dtype

    def zero_grad(self):
        self.grad.fill(0)


class ParamBlock:
    __slots__ = ("name", "var", "learnable")

    def __init__(self, name, var, learnable=True):
        self.name, self.var, self.learnable = name, var, learnable

    def __repr__(self):
        return f"ParamBlock({self.name!r}, shape={self.var.shape}, learnable={self.learnable})"


@dataclass
class ModelConfig:
    vocab_size: int
    embedding_size: int = 512
    hidden_size: int = 512
    depth: int = 2
    dropout: float = 0.2
    output_tanh: bool = True
    shared_embeddings: bool = False

    def validate(self):
        for f in ("vocab_size", "embedding_size", "hidden_size", "depth"):
            if getattr(self, f) < 1:
                raise ConfigError(f"{f} must be positive, got {getattr(self, f)}")
        if not 0.0 <= self.dropout < 1.0:
            raise ConfigError(f"dropout must be in [0, 1), got {self.dropout}")
        return self


def block_layout(cfg: ModelConfig):
    """[(name, (rows, cols), kind)] in registry order; kind drives init.

    kind: "w" uniform(+-0.1) draw, "b0" zeros, "b1" ones (forget bias).
    """
    V, E, H, L = cfg.vocab_size, cfg.embedding_size, cfg.hidden_size, cfg.depth
    out = [("src_embed", (V, E), "w")]
    if not cfg.shared_embeddings:
        out.append(("tgt_embed", (V, E), "w"))

    def lstm(prefix, din):
        ws = [(f"{prefix}.w_{g}", (din + H, H), "w") for g in GATES]
        bs = [(f"{prefix}.b_{g}", (H, 1), "b1" if g == "f" else "b0") for g in GATES]
        return ws + bs

    out += lstm("enc.l1.fwd", E) + lstm("enc.l1.bwd", E)
    for k in range(2, L + 1):
        out += lstm(f"enc.l{k}", H)
    for k in range(1, L + 1):
        out += lstm(f"dec.l{k}", E if k == 1 else H)
    out += [("att.w_a.w", (H, H), "w"), ("att.w_c.w", (2 * H, H), "w"),
            ("out.w", (H, V), "w"), ("out.b", (V, 1), "b0")]
    return out


class ModelParams:
    """Every trainable block in declaration order; init draws in that order."""

    def __init__(self, config: ModelConfig, rng: Rng, dtype=None):
        config.validate()
        self.dtype = np.dtype(dtype or np.float32)
        self._registry = []
        for name, shape, kind in block_layout(config):
            if kind == "w":
                data = rng.uniform(-INIT_SCALE, INIT_SCALE, shape, dtype=self.dtype)
            else:
                data = np.full(shape, 1.0 if kind == "b1" else 0.0, dtype=self.dtype)
            self._registry.append(ParamBlock(name, Variable(data)))
        self._by_name = {b.name: b for b in self._registry}

    def blocks(self):
        return list(self._registry)

    def __getitem__(self, name):
        return self._by_name[name]

    def zero_grads(self):
        for b in self._registry:
            b.var.zero_grad()

    def copy_data(self):
        return {b.name: b.var.data.copy() for b in self._registry}

    def load_data(self, snapshot):
        for b in self._registry:
            if b.name not in snapshot:
                raise ConfigError(f"snapshot is missing parameter {b.name!r}")
            if snapshot[b.name].shape != b.var.shape:
                raise ShapeError(f"snapshot shape {snapshot[b.name].shape} != {b.var.shape} for {b.name!r}")
            np.copyto(b.var.data, snapshot[b.name].astype(self.dtype))


class Model:
    def __init__(self, config: ModelConfig, params: ModelParams):
        self.config = config
        self.params = params

    @classmethod
    def new(cls, config: ModelConfig, rng: Rng, dtype=None) -> "Model":
        return cls(config, ModelParams(config, rng, dtype=dtype))


@dataclass
class TrainConfig:
    learning_rate: float = 1.0
    decay_factor: float = 0.7
    label_smoothing: float = 0.1
    patience: int = 12
    eval_interval_sentences: int = 400_000
    max_bad_decays: int = 2
    grad_clip_norm: float | None = 5.0
    batch_size: int = 64
    max_len: int = 100
    max_epochs: int | None = None
    seed: int = 1


@dataclass
class Batch:
    src_ids: np.ndarray
    tgt_ids: np.ndarray
    src_mask: np.ndarray
    tgt_mask: np.ndarray
    src_lengths: list = field(default_factory=list)
    tgt_lengths: list = field(default_factory=list)
    indices: list = field(default_factory=list)
