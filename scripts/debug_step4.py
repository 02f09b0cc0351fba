"""Poison freed device memory with NaN, then check each bf16 forward kernel
against a torch recomputation from its own (dumped) inputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import minmt_oracle as O  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from tests.gpu_helpers import cfg_of, scaled_params  # noqa: E402

V, E, H, L, B, S, T = (1000, 128, 128, 1, 16, 9, 8)
d = O.Dims(V, E, H, L, 0.0)
params = scaled_params(d, 3, 0.1)
src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=4, ragged=True)
NT, NS = B * T, B * S
poison = os.environ.get("POISON", "1") == "1"
if poison:
    x = torch.full((3 << 28,), float("nan"), device="cuda")
    torch.cuda.synchronize()
    del x
    torch.cuda.empty_cache()
eng = Engine(cfg_of(d), mode="bf16")
eng.upload(params)
eng.set_option("stop_after", 1)
eng.stage(src, sm, tgt, tm)
eng.run(1.0, 5.0, 0.1, None, update=False)
bf = lambda a: torch.tensor(a).bfloat16().float()  # noqa: E731
Y = eng.debug_buffer("Y").reshape(NT, V)
hod = eng.debug_buffer("hod").reshape(NT, H)
ho = eng.debug_buffer("ho").reshape(NT, H)
cst = eng.debug_buffer("cst_att").reshape(NT, 2 * H)
u = eng.debug_buffer("u_att").reshape(NT, H)
yd = eng.debug_buffer(f"yext:{2 * L}").reshape(T + 1, B, H)[1:].reshape(NT, H)
for name, arr in [("Y", Y), ("hod", hod), ("ho", ho), ("cst", cst), ("u", u), ("ydec", yd)]:
    print(name, "nan", int(np.isnan(arr).sum()), "max", float(np.nanmax(np.abs(arr))))
ref_Y = torch.tanh(torch.tensor(hod) @ bf(params["out.w"]) + torch.tensor(params["out.b"][:, 0])).numpy()
print("Y vs tanh(hod Wo + b)", O.norm_rel_err(Y, ref_Y))
ref_ho = torch.tanh(torch.tensor(cst) @ bf(params["att.w_c.w"])).numpy()
print("ho vs tanh(cst Wc)", O.norm_rel_err(ho, ref_ho))
ref_u = (torch.tensor(yd) @ bf(params["att.w_a.w"])).numpy()
print("u vs Ht Wa", O.norm_rel_err(u, ref_u))
print("cst[:,H:] vs Ht", O.norm_rel_err(cst[:, H:], yd))
print("hod vs bf16(ho)", O.norm_rel_err(hod, bf(ho).numpy()))
eng.close()

# error pattern + repeat + hook on identical data
err = np.abs(Y - ref_Y)
print("err by 128-row/256-col tile:")
for n0 in range(0, V, 256):
    print("  cols", n0, "max err %.3e" % err[:, n0:n0 + 256].max(), "rows bad", int((err[:, n0:n0 + 256].max(axis=1) > 1e-3).sum()))
print("worst rows", np.argsort(-err.max(axis=1))[:10].tolist(), "worst cols", np.argsort(-err.max(axis=0))[:10].tolist())
from paper_1802_07170_b200 import _lib  # noqa: E402
lib = _lib.load()
A = torch.tensor(hod).bfloat16().cuda().contiguous()
Bm = bf(params["out.w"]).bfloat16().cuda().contiguous()
for bn in (128, 256):
    C = torch.zeros(NT, V).cuda()
    lib.cmt_test_gemm(1, NT, V, H, A.data_ptr(), H, 0, Bm.data_ptr(), V, 1, C.data_ptr(), V, bn, 0, None)
    print("hook bn", bn, O.norm_rel_err(np.tanh(C.cpu().numpy() + params["out.b"][:, 0]), ref_Y))
eng = Engine(cfg_of(d), mode="bf16")
eng.upload(params)
eng.set_option("stop_after", 1)
eng.stage(src, sm, tgt, tm)
for i in range(4):
    eng.run(1.0, 5.0, 0.1, None, update=False)
    Y2 = eng.debug_buffer("Y").reshape(NT, V)
    print("engine repeat", i, "%.3e" % O.norm_rel_err(Y2, ref_Y), "vs first %.3e" % O.norm_rel_err(Y2, Y))
