import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_07170_b200 import _lib  # noqa: E402

lib = _lib.load()


def gemm_ld(M, N, K, am, bm, bn):
    g = torch.Generator().manual_seed(0)
    Al = torch.randn(M, K, generator=g).bfloat16()
    Bl = torch.randn(N, K, generator=g).bfloat16()
    A = (Al.t().contiguous() if am else Al.contiguous()).cuda()
    B = (Bl.t().contiguous() if bm else Bl.contiguous()).cuda()
    C = torch.zeros(M, N).cuda()
    rc = lib.cmt_test_gemm(1, M, N, K, A.data_ptr(), M if am else K, am, B.data_ptr(), N if bm else K, bm,
                           C.data_ptr(), N, bn, 0, None)
    ref = Al.float() @ Bl.float().t()
    return rc, ((C.cpu() - ref).abs().max() / ref.abs().max()).item()


for sh in [(320, 1000, 128, 0, 1, 128), (320, 1000, 128, 0, 1, 256), (320, 128, 1000, 0, 0, 128),
           (256, 128, 320, 1, 1, 128), (128, 1000, 320, 1, 1, 256), (128, 1000, 320, 1, 1, 128),
           (320, 512, 128, 0, 1, 256), (16, 512, 128, 0, 1, 64), (16, 128, 512, 0, 0, 64),
           (128, 512, 320, 1, 1, 256), (320, 128, 512, 0, 0, 128), (320, 256, 128, 0, 0, 256),
           (320, 128, 128, 0, 1, 128), (320, 128, 256, 0, 1, 128)]:
    print(sh, gemm_ld(*sh), flush=True)

from oracle import minmt_oracle as O  # noqa: E402
from tests.gpu_helpers import engine_step, oracle_step, scaled_params  # noqa: E402

for case in [(1000, 128, 128, 1, 16, 9, 8), (256, 128, 128, 1, 16, 20, 20), (256, 128, 128, 1, 16, 20, 8),
             (256, 128, 128, 1, 16, 9, 20), (256, 128, 128, 1, 8, 20, 20), (64, 32, 32, 2, 8, 7, 6)]:
    V, E, H, L, B, S, T = case
    d = O.Dims(V, E, H, L, 0.2)
    params = scaled_params(d, 3, 0.1)
    batch = O.synthetic_batch(V, S, T, B, seed=4, ragged=True)
    ol, _, og, _, _ = oracle_step(d, params, batch, 0.1, 1.0, 5.0, 21, update=False)
    try:
        loss, _, g, _, _ = engine_step(d, params, batch, 0.1, 1.0, 5.0, 21, "bf16", update=False)
    except Exception as e:
        print(case, "EXC", e)
        continue
    errs = {n: O.norm_rel_err(g[n], og[n]) for n in g}
    bad = {n: "%.1e" % e for n, e in errs.items() if e > 2e-2}
    print(case, "loss", loss, ol, "worst", "%.2e" % max(errs.values()), list(bad.items())[:6], flush=True)
