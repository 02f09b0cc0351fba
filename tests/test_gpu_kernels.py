"""Per-kernel GPU parity: the tcgen05 GEMM in every operand layout the step
uses (vs a torch fp32 matmul of the same bf16 operands) and the PCG64 dropout
kernel (vs numpy's Generator.random, bit-exact)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1802_07170_b200 import _lib  # noqa: E402


def _gemm(mode, M, N, K, a_mn, b_mn, bn, beta=0, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    dt = torch.bfloat16 if mode == _lib.MODE_BF16 else torch.float32
    Al = torch.randn(M, K, generator=g).to(dt)
    Bl = torch.randn(N, K, generator=g).to(dt)
    # physical layouts: K-major stores [rows][K]; MN-major stores [K][rows]
    A = (Al.t().contiguous() if a_mn else Al.contiguous()).cuda()
    B = (Bl.t().contiguous() if b_mn else Bl.contiguous()).cuda()
    C0 = torch.randn(M, N, generator=g)
    C = C0.clone().cuda()
    lda = M if a_mn else K
    ldb = N if b_mn else K
    lib = _lib.load()
    rc = lib.cmt_test_gemm(mode, M, N, K, A.data_ptr(), lda, a_mn, B.data_ptr(), ldb, b_mn, C.data_ptr(), N, bn, beta, None)
    assert rc == 0, lib.cmt_last_error(None)
    ref = Al.float() @ Bl.float().t() + (C0 if beta else 0)
    return C.cpu(), ref


@pytest.mark.parametrize("a_mn,b_mn", [(0, 1), (0, 0), (1, 1)])
@pytest.mark.parametrize("bn", [64, 128, 256, 129, 257])  # 129/257: CTA-pair (cta_group::2) 256-row tiles
@pytest.mark.parametrize("shape", [(128, 256, 64), (300, 520, 200), (1000, 1100, 1024), (64, 96, 40)])
def test_tcgen05_gemm_layouts(a_mn, b_mn, bn, shape):
    M, N, K = shape
    if (a_mn or b_mn) and (M % 8 or N % 8):
        pytest.skip("MN-major needs 16-byte aligned rows")
    if (not a_mn and K % 8) or (not b_mn and K % 8):
        pytest.skip("K-major needs 16-byte aligned rows")
    C, ref = _gemm(_lib.MODE_BF16, M, N, K, a_mn, b_mn, bn)
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err  # bf16 inputs are exact in both; only fp32 summation order differs


@pytest.mark.parametrize("bn", [256, 257])
def test_tcgen05_gemm_accumulate_and_many_tiles(bn):
    C, ref = _gemm(_lib.MODE_BF16, 6400, 2048, 1024, 0, 1, bn, beta=1, seed=3)
    assert (C - ref).abs().max().item() / ref.abs().max().item() < 1e-5


@pytest.mark.parametrize("a_mn,b_mn", [(0, 1), (0, 0), (1, 1)])
def test_fp32_simt_gemm_layouts(a_mn, b_mn):
    C, ref = _gemm(_lib.MODE_FP32, 77, 130, 45, a_mn, b_mn, 64)
    assert (C - ref).abs().max().item() / ref.abs().max().item() < 1e-6


@pytest.mark.parametrize("N,H,base,p", [(100, 48, 0, 0.2), (6400, 1024, 123456789, 0.3), (37, 8, 5, 0.5)])
def test_dropout_kernel_matches_numpy_pcg64(N, H, base, p):
    from paper_1802_07170_b200.engine import pcg_state
    gen = np.random.Generator(np.random.PCG64(77))
    sh, sl, ih, il = pcg_state(gen)
    x = torch.randn(N, H).cuda()
    y = torch.empty_like(x)
    keep = torch.empty(N, H, dtype=torch.uint8, device="cuda")
    lib = _lib.load()
    assert lib.cmt_test_dropout(sh, sl, ih, il, base, N, H, p, x.data_ptr(), y.data_ptr(), keep.data_ptr()) == 0
    gen.bit_generator.advance(base)
    u = gen.random(size=(H, N))             # reference draw layout: (H, N) C order
    ref_keep = (u >= p).T
    assert np.array_equal(keep.cpu().numpy().astype(bool), ref_keep)
    scale = np.float32(1.0) / np.float32(1.0 - p)
    ref_y = x.cpu().numpy() * (ref_keep.astype(np.float32) * scale)
    assert np.array_equal(y.cpu().numpy(), ref_y)


@pytest.mark.parametrize("bn", [128, 256, 257])
@pytest.mark.parametrize("shape", [(6400, 1000, 256), (300, 520, 200)])
def test_tcgen05_gemm_bias_tanh_bf16_out(bn, shape):
    """The logits epilogue: C = bf16(tanh(A B^T + bias)), via the TMA-store path."""
    M, N, K = shape
    g = torch.Generator(device="cpu").manual_seed(7)
    Al = (0.05 * torch.randn(M, K, generator=g)).to(torch.bfloat16)
    Bw = (0.05 * torch.randn(K, N, generator=g)).to(torch.bfloat16)  # MN-major weight (dim_in, dim_out)
    bias = 0.1 * torch.randn(N, generator=g)
    A, B, bd = Al.cuda(), Bw.cuda(), bias.cuda()
    C = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    lib = _lib.load()
    rc = lib.cmt_test_gemm(_lib.MODE_BF16, M, N, K, A.data_ptr(), K, 0, B.data_ptr(), N, 1, C.data_ptr(), N, bn,
                           2 | 4, bd.data_ptr())
    assert rc == 0, lib.cmt_last_error(None)
    ref = torch.tanh(Al.float() @ Bw.float() + bias)
    err = (C.float().cpu() - ref).abs().max().item()
    assert err < 1.5e-2 * max(1.0, ref.abs().max().item()), err  # bf16 output rounding + tanh.approx


@pytest.mark.parametrize("beta", [0, 1])
@pytest.mark.parametrize("bn", [256, 257])
def test_tcgen05_gemm_split_k(beta, bn):
    """dX-shaped GEMM (M=6400, N=1024, K=4096): the launcher splits K and the
    slices TMA-reduce-add into C (zeroed first unless accumulating)."""
    C, ref = _gemm(_lib.MODE_BF16, 6400, 1024, 4096, 0, 0, bn, beta=beta, seed=5)
    assert (C - ref).abs().max().item() / ref.abs().max().item() < 1e-5


def test_tcgen05_gemm_stream_k_deterministic():
    """dW-shaped GEMM (M=1024, N=4096, K=6400: 64 pair tiles < 74 pairs) with
    owner/helper stream-K enabled (two pieces per tile reduce-added into zeroed
    C): correct and bit-identical across runs."""
    lib = _lib.load()
    assert lib.cmt_set_option(None, b"splitk", 3) == 0
    try:
        C1, ref = _gemm(_lib.MODE_BF16, 1024, 4096, 6400, 1, 1, 257, seed=9)
        assert (C1 - ref).abs().max().item() / ref.abs().max().item() < 1e-5
        C2, _ = _gemm(_lib.MODE_BF16, 1024, 4096, 6400, 1, 1, 257, seed=9)
        assert torch.equal(C1, C2)
    finally:
        assert lib.cmt_set_option(None, b"splitk", 1) == 0
