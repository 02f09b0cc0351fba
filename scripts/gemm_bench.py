"""Micro-benchmark of the tcgen05 GEMM family on the c3 step's shapes.

    python scripts/gemm_bench.py [--only NAME] [--iters N]

Times each (shape, tile) with CUDA events on the launch stream (the test hook
synchronises after every launch, so each launch is timed alone).  Prints
TFLOP/s per configuration."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_07170_b200 import _lib  # noqa: E402

# name: (M, N, K, a_mn, b_mn, flags)  flags: 1 beta, 2 bf16 out, 4 tanh, 8 no bias
SHAPES = {
    "logits": (6400, 50000, 1024, 0, 1, 2 | 4),        # tanh(H_o W_o + b_o), bf16 out
    "logits_nobias": (6400, 50000, 1024, 0, 1, 2 | 4 | 8),   # epilogue ablations (8: no bias)
    "logits_notanh": (6400, 50000, 1024, 0, 1, 2),
    "logits_plain": (6400, 50000, 1024, 0, 1, 2 | 8),
    "logits_f32": (6400, 50000, 1024, 0, 1, 0),
    "dWo": (1024, 50000, 6400, 1, 1, 0),               # H_o^T dY
    "dHo": (6400, 1024, 50000, 0, 0, 2),               # dY W_o^T
    "ux": (6400, 4096, 1024, 0, 1, 0),                 # X W_x + b (hoisted input projection)
    "dWx": (1024, 4096, 6400, 1, 1, 0),                # X^T dU
    "dX": (6400, 1024, 4096, 0, 0, 0),                 # dU W_x^T
    "dWx75": (1024, 3072, 6400, 1, 1, 0),              # the main-stream 75 % of a level's dW columns
    # c2 (2x512, V=30k, B=64, S=T=50): K = 512 products
    "logits_c2": (3200, 30000, 512, 0, 1, 2 | 4),
    "logits_c2_plain": (3200, 30000, 512, 0, 1, 2 | 8),
    "dWo_c2": (512, 30000, 3200, 1, 1, 0),
    "dHo_c2": (3200, 512, 30000, 0, 0, 2),
    "ux_c2": (3200, 2048, 512, 0, 1, 0),
    "dWx_c2": (512, 2048, 3200, 1, 1, 0),
    "dX_c2": (3200, 512, 2048, 0, 0, 0),
}


def run(name, tiles, iters):
    M, N, K, a_mn, b_mn, flags = SHAPES[name]
    g = torch.Generator(device="cpu").manual_seed(0)
    A = torch.randn((K, M) if a_mn else (M, K), generator=g).to(torch.bfloat16).cuda()
    B = torch.randn((K, N) if b_mn else (N, K), generator=g).to(torch.bfloat16).cuda()
    C = torch.zeros(M, N, dtype=torch.bfloat16 if flags & 2 else torch.float32, device="cuda")
    bias = torch.zeros(N, device="cuda")
    use_bias = not (flags & 8)
    flags &= 7
    lda = M if a_mn else K
    ldb = N if b_mn else K
    lib = _lib.load()
    out = []
    for bn in tiles:
        def call():
            rc = lib.cmt_test_gemm(_lib.MODE_BF16, M, N, K, A.data_ptr(), lda, a_mn, B.data_ptr(), ldb, b_mn,
                                   C.data_ptr(), N, bn, flags, bias.data_ptr() if use_bias else None)
            assert rc == 0, lib.cmt_last_error(None)
        call()
        ts = []
        for _ in range(iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            call()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        tf = 2.0 * M * N * K / (ms / 1e3) / 1e12
        out.append((bn, ms, tf))
        print(f"{name:8s} M={M:6d} N={N:6d} K={K:6d} tile={'%d%s' % (bn - (bn & 1), 'x2' if bn & 1 else ''):6s} "
              f"{ms * 1e3:9.1f} us  {tf:7.1f} TFLOP/s", flush=True)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--iters", type=int, default=7)
    ap.add_argument("--tiles", default="128,256,129,257")
    ap.add_argument("--opt", type=int, default=None, help="engine gemm_opt bits (1: natural K order, 2: N-fastest)")
    ap.add_argument("--splitk", type=int, default=None, help="engine splitk bits (1 split-K 2, 2 owner/helper, 4 stream-K)")
    a = ap.parse_args()
    if a.opt is not None:
        assert _lib.load().cmt_set_option(None, b"gemm_opt", a.opt) == 0
    if a.splitk is not None:
        assert _lib.load().cmt_set_option(None, b"splitk", a.splitk) == 0
    tiles = [int(x) for x in a.tiles.split(",")]
    for n in SHAPES:
        if a.only and n not in a.only.split(","):
            continue
        run(n, tiles, a.iters)
