"""Data parallelism over sentence batches.

The step is exactly data-parallel: no op couples batch columns, so each rank
runs the full step on its own column shard.  Two host-side facts make the sum
of shard gradients equal the reference gradient of the concatenated batch:

* every rank scales its CE gradient by 1 / global_ntok, where global_ntok is
  the float32 sum of tgt_mask over ALL ranks (training.py:108-119 divides by
  the batch's token count), and
* the engine all-reduces (NCCL, sum) the dense gradients, the loss sum and the
  error status inside the step, before the global-norm clip and the update,
  so every rank applies the identical update (training.py:123-142);
* the embedding gradients are row-sparse: each rank stages only the rows its
  shard touches, the ranks agree on the union of those ids on the host
  (``exchange_rows``, before the step) and the engine all-reduces and updates
  just the union rows (rows outside it have zero gradient in every rank).

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


def _load_torch_nccl():
    """Import torch before the engine first touches NCCL: the engine then binds
    the libnccl.so.2 torch links (already in the process) instead of loading
    another copy under the same soname, which a later torch import would reuse."""
    import torch  # noqa: F401


def nccl_unique_id() -> bytes:
    _load_torch_nccl()
    buf = ctypes.create_string_buffer(128)
    lib = _lib.load()
    rc = lib.cmt_nccl_unique_id(buf)
    if rc:
        raise RuntimeError(lib.cmt_last_error(None).decode())
    return buf.raw


def attach(engine, dist, rank, world):
    """Create the engine's NCCL communicator (rank 0's unique id broadcast via torch.distributed)."""
    _load_torch_nccl()
    obj = [nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    uid = ctypes.create_string_buffer(obj[0], 128)
    engine._check(engine.lib.cmt_set_comm(engine.h, uid, rank, world))


def union_rows(id_lists):
    """Ascending union of several ascending id arrays (the rows any rank touches)."""
    if not id_lists:
        return np.empty(0, dtype=np.int32)
    return np.unique(np.concatenate([np.asarray(x, dtype=np.int32) for x in id_lists])).astype(np.int32)


def gather_ids(ids, dist):
    """All ranks' id arrays (variable lengths) via torch.distributed all_gather."""
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    n = torch.tensor([len(ids)], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(dist.get_world_size())]
    dist.all_gather(sizes, n)
    mx = int(max(int(x.item()) for x in sizes))
    buf = torch.full((max(mx, 1),), -1, dtype=torch.int32, device=dev)
    buf[:len(ids)] = torch.as_tensor(np.asarray(ids, dtype=np.int32), device=dev)
    out = [torch.empty_like(buf) for _ in range(dist.get_world_size())]
    dist.all_gather(out, buf)
    return [o[:int(s.item())].cpu().numpy() for o, s in zip(out, sizes)]


def exchange_rows(engine, dist):
    """Give the engine the union of every rank's staged embedding rows (per table)."""
    for t in range(engine.n_tables):
        engine.set_union(t, union_rows(gather_ids(engine.staged_rows(t), dist)))
