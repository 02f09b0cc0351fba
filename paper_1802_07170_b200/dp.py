"""Data parallelism over sentence batches.

The step is exactly data-parallel: no op couples batch columns, so each rank
runs the full step on its own column shard.  Two host-side facts make the sum
of shard gradients equal the reference gradient of the concatenated batch:

* every rank scales its CE gradient by 1 / global_ntok, where global_ntok is
  the float32 sum of tgt_mask over ALL ranks (training.py:108-119 divides by
  the batch's token count), and
* the engine all-reduces (NCCL, sum) the dense gradients, the loss sum and the
  error status inside the step, before the global-norm clip and the update,
  so every rank applies the identical update (training.py:123-142).

Dropout draws are per rank (each rank's own PCG64 stream); the single-process
reference equality holds at dropout 0.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def shard_columns(arrays, rank, world):
    """Contiguous column block of each (steps, B) array for this rank."""
    B = np.shape(arrays[0])[1]
    if B % world:
        raise ValueError(f"global batch {B} is not divisible by world size {world}")
    b = B // world
    return [np.ascontiguousarray(np.asarray(a)[:, rank * b:(rank + 1) * b]) for a in arrays]


def global_ntok(tgt_mask, dist=None):
    """float32 token count of this rank's shard, summed over ranks."""
    local = float(np.asarray(tgt_mask, dtype=np.float32).sum(dtype=np.float32))
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([local], dtype=torch.float64, device=dev)
    dist.all_reduce(t)
    return float(t.item())


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    lib = _lib.load()
    rc = lib.cmt_nccl_unique_id(buf)
    if rc:
        raise RuntimeError(lib.cmt_last_error(None).decode())
    return buf.raw


def attach(engine, dist, rank, world):
    """Create the engine's NCCL communicator (rank 0's unique id broadcast via torch.distributed)."""
    obj = [nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    uid = ctypes.create_string_buffer(obj[0], 128)
    engine._check(engine.lib.cmt_set_comm(engine.h, uid, rank, world))
