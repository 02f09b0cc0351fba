"""B200-native CytonMT train-step engine (drop-in for minmt.training.train_step).

Host-side mirror of the reference types lives in ``model``; the CUDA engine is
``libcytonb200.so`` (C ABI: include/cytonmt_b200.h) bound by ``engine``;
``training.train_step`` is the drop-in.
"""

from .model import Batch, Model, ModelConfig, ModelParams, Rng, TrainConfig  # noqa: F401

__all__ = ["Batch", "Model", "ModelConfig", "ModelParams", "Rng", "TrainConfig"]
