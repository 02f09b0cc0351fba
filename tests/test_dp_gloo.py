"""Data-parallel host logic on CPU with a real 2-rank gloo process group.

Each rank takes its column shard of the global batch (dp.shard_columns),
computes the global token count by all-reduce (dp.global_ntok), runs the
oracle step on its shard with the CE gradient normalised by the GLOBAL token
count, and the ranks sum gradients and loss — exactly what the engine does
with NCCL inside the step.  The summed gradients, loss and clipped-SGD update
must equal the single-process reference on the concatenated batch.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import minmt_oracle as O

D = O.Dims(53, 8, 16, 2, 0.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _params():
    return O.init_params(D, np.random.default_rng(7))


def _batch():
    return O.synthetic_batch(D.vocab, 6, 5, 8, seed=3, ragged=True)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1802_07170_b200 import dp
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        src, sm, tgt, tm = dp.shard_columns(_batch(), rank, world)
        gnt = dp.global_ntok(tm, dist)
        p = _params()
        loss, g, _ = O.forward_backward(p, D, src, sm, tgt, tm, 0.1)
        names = [n for n, _ in O.registry(D)]
        local = float(tm.sum(dtype=np.float32))
        flat = torch.from_numpy(np.concatenate([g[n].ravel().astype(np.float64) * (local / gnt) for n in names]))
        dist.all_reduce(flat)
        lsum = torch.tensor([loss * local], dtype=torch.float64)
        dist.all_reduce(lsum)
        # identical clipped update on every rank from the summed grads
        gsum, off = {}, 0
        for n, s in O.registry(D):
            k = int(np.prod(s))
            gsum[n] = flat[off:off + k].numpy().reshape(s).astype(np.float32)
            off += k
        norm = O.sgd_step(p, gsum, names, 1.0, 0.05)
        q.put((rank, flat.numpy(), float(lsum.item() / gnt), gnt, norm, {n: p[n] for n in names}))
    finally:
        dist.destroy_process_group()


def test_dp_two_rank_gloo_sum_equals_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    # every rank holds the same reduced state
    assert np.array_equal(res[0][1], res[1][1]) and res[0][2] == res[1][2]
    src, sm, tgt, tm = _batch()
    p = _params()
    loss, g, _ = O.forward_backward(p, D, src, sm, tgt, tm, 0.1)
    names = [n for n, _ in O.registry(D)]
    ref = np.concatenate([g[n].ravel().astype(np.float64) for n in names])
    assert res[0][3] == float(tm.sum())
    assert abs(res[0][2] - loss) <= 1e-6 * loss
    assert O.norm_rel_err(res[0][1], ref) < 1e-5
    norm = O.sgd_step(p, g, names, 1.0, 0.05)
    assert abs(res[0][4] - norm) <= 1e-5 * norm
    for n in names:
        assert O.norm_rel_err(res[0][5][n], p[n]) < 1e-6, n


def test_shard_columns_and_errors():
    from paper_1802_07170_b200 import dp
    a = np.arange(24).reshape(3, 8)
    s0, = dp.shard_columns([a], 0, 4)
    s3, = dp.shard_columns([a], 3, 4)
    assert s0.tolist() == [[0, 1], [8, 9], [16, 17]] and s3[:, 1].tolist() == [7, 15, 23]
    with pytest.raises(ValueError):
        dp.shard_columns([a], 0, 3)
    assert dp.global_ntok(np.ones((3, 2), np.float32)) == 6.0


def _rows_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1802_07170_b200 import dp
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        # each rank's staged rows: the ascending unique ids of its shard (the
        # engine's cmt_staged_rows), different lengths per rank
        src, sm, tgt, tm = dp.shard_columns(_batch(), rank, world)
        mine = np.unique(src[sm > 0]).astype(np.int32) if rank == 0 else np.array([0, 5, 52], np.int32)
        got = dp.union_rows(dp.gather_ids(mine, dist))
        q.put((rank, mine, got))
    finally:
        dist.destroy_process_group()


def test_dp_rows_union_exchange_two_ranks():
    """dp.exchange_rows' host side (gather_ids + union_rows) on a real 2-rank
    gloo group: every rank obtains the same ascending union of all ranks'
    staged embedding rows (what the engine all-reduces and updates)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = np.unique(np.concatenate([res[0][1], res[1][1]]))
    for r in res:
        assert r[2].dtype == np.int32 and np.array_equal(r[2], expect)
    assert np.all(np.diff(expect) > 0)
