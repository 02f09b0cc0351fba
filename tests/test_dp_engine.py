"""Two-rank data-parallel engine test (NCCL over NVLink); skipped unless two
GPUs are visible.  Each rank runs the engine on its column shard of the global
batch (global token count, NCCL all-reduce of dense gradient buckets during
the backward, the embedding rows union, flag-wise status) and must end with
the parameters of ONE engine stepping on the concatenated batch (dropout 0:
the draws are per rank), SURVEY §8(e)."""

import os
import socket

import numpy as np
import pytest

from oracle import minmt_oracle as O

pytestmark = pytest.mark.gpu

D = O.Dims(304, 64, 256, 2, 0.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    from tests.gpu_helpers import scaled_params
    return scaled_params(D, 5, 0.1), O.synthetic_batch(D.vocab, 9, 7, 16, seed=4, ragged=True)


def _worker(rank, world, port, mode, q):
    import torch
    import torch.distributed as dist

    from paper_1802_07170_b200 import dp
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    from tests.gpu_helpers import cfg_of
    torch.cuda.set_device(rank)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        params, batch = _setup()
        src, sm, tgt, tm = dp.shard_columns(batch, rank, world)
        eng = Engine(cfg_of(D), mode=mode, device=rank)
        eng.upload(params)
        eng.set_dp(dist, rank, world)
        gnt = dp.global_ntok(tm, dist)
        eng._stage_batch(Batch(src, tgt, sm, tm), None)
        r = eng.run(1.0, 0.05, 0.1, None, global_ntok=gnt)
        q.put((rank, r.loss_sum, r.grad_norm, eng.params()))
        eng.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_two_rank_engine_equals_one_rank_on_full_batch(mode):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    from paper_1802_07170_b200.engine import Engine
    from paper_1802_07170_b200.model import Batch
    from tests.gpu_helpers import cfg_of
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    params, (src, sm, tgt, tm) = _setup()
    eng = Engine(cfg_of(D), mode=mode)
    eng.upload(params)
    loss, norm = eng.step(Batch(src, tgt, sm, tm), 1.0, 0.05, 0.1, None)
    ref = eng.params()
    eng.close()
    tol = 1e-5 if mode == "fp32" else 1e-3
    for rank, lsum, gnorm, p in res:
        assert abs(lsum / float(tm.sum()) - loss) <= tol * loss, rank
        assert abs(gnorm - norm) <= tol * norm, rank
        for n in ref:
            assert O.norm_rel_err(p[n], ref[n]) < tol, (rank, n)
    for n in ref:  # every rank applied the identical update
        assert np.array_equal(res[0][3][n], res[1][3][n]), n
