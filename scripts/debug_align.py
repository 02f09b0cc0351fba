"""Is the tcgen05 GEMM sensitive to operand base-address alignment?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_07170_b200 import _lib  # noqa: E402

lib = _lib.load()
torch.manual_seed(0)


def run(M, N, K, am, bm, bn, offA, offB, offC, flags):
    Al = torch.randn(M, K).bfloat16()
    Bl = torch.randn(N, K).bfloat16()
    bias = torch.randn(N).cuda()
    A0 = (Al.t().contiguous() if am else Al.contiguous()).reshape(-1)
    B0 = (Bl.t().contiguous() if bm else Bl.contiguous()).reshape(-1)
    Abuf = torch.zeros(A0.numel() + 4096, dtype=torch.bfloat16, device="cuda")
    Bbuf = torch.zeros(B0.numel() + 4096, dtype=torch.bfloat16, device="cuda")
    Abuf[offA // 2: offA // 2 + A0.numel()] = A0.cuda()
    Bbuf[offB // 2: offB // 2 + B0.numel()] = B0.cuda()
    cdt = torch.bfloat16 if flags & 2 else torch.float32
    Cbuf = torch.zeros(M * N + 4096, dtype=cdt, device="cuda")
    esz = 2 if flags & 2 else 4
    C = Cbuf[offC // esz: offC // esz + M * N]
    rc = lib.cmt_test_gemm(1, M, N, K, Abuf.data_ptr() + offA, M if am else K, am, Bbuf.data_ptr() + offB,
                           N if bm else K, bm, C.data_ptr(), N, bn, flags, bias.data_ptr())
    ref = Al.float() @ Bl.float().t() + bias.cpu()
    if flags & 4:
        ref = torch.tanh(ref)
    got = C.float().cpu().reshape(M, N)
    return rc, ((got - ref).abs().max() / ref.abs().max()).item()


fails = 0
for shape in [(128, 1000, 128), (320, 1000, 128), (128, 512, 128), (256, 1000, 256)]:
    for (am, bm) in [(0, 1), (0, 0), (1, 1)]:
        for bn in (128, 256):
            for offA in (0, 16, 128, 256, 512):
                for offB in (0, 16, 128, 256, 512):
                    for flags in (0, 6):
                        rc, err = run(*shape, am, bm, bn, offA, offB, 256, flags)
                        tol = 1e-2 if flags & 2 else 1e-5
                        if rc or err > tol:
                            fails += 1
                            print("FAIL", shape, am, bm, bn, offA, offB, flags, rc, "%.3e" % err, flush=True)
print("fails", fails)
