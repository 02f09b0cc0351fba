import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import minmt_oracle as O  # noqa: E402
from paper_1802_07170_b200 import _lib  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from tests.gpu_helpers import cfg_of, scaled_params  # noqa: E402

lib = _lib.load()
V, E, H, L, B, S, T = (1000, 128, 128, 1, 16, 9, 8)
d = O.Dims(V, E, H, L, 0.0)
params = scaled_params(d, 3, 0.1)
src, sm, tgt, tm = O.synthetic_batch(V, S, T, B, seed=4, ragged=True)
NT = B * T
eng = Engine(cfg_of(d), mode="bf16")
eng.upload(params)
eng.set_option("stop_after", 1)
eng.stage(src, sm, tgt, tm)
eng.run(1.0, 5.0, 0.1, None, update=False)
Y = eng.debug_buffer("Y").reshape(NT, V)
hod = eng.debug_buffer("hod").reshape(NT, H)
wo = torch.tensor(params["out.w"]).bfloat16().float()
bo = torch.tensor(params["out.b"][:, 0])
ref = torch.tanh(torch.tensor(hod) @ wo + bo).numpy()
print("engine Y vs torch(hod@Wo_bf16)", O.norm_rel_err(Y, ref))
rows_bad = np.where(np.abs(Y - ref).max(axis=1) > 1e-3)[0]
cols_bad = np.where(np.abs(Y - ref).max(axis=0) > 1e-3)[0]
print("bad rows", len(rows_bad), rows_bad[:40].tolist())
print("bad cols", len(cols_bad), cols_bad[:10].tolist(), cols_bad[-10:].tolist())
# same GEMM through the isolated hook, fp32 C
A = torch.tensor(hod).bfloat16().cuda().contiguous()
Bm = wo.bfloat16().cuda().contiguous()  # [H][V] = MN-major B
for bn in (128, 256):
    C = torch.zeros(NT, V).cuda()
    rc = lib.cmt_test_gemm(1, NT, V, H, A.data_ptr(), H, 0, Bm.data_ptr(), V, 1, C.data_ptr(), V, bn, 0, None)
    print("hook bn", bn, rc, O.norm_rel_err(C.cpu().numpy(), (torch.tensor(hod) @ wo).numpy()))
# repeat engine forward twice more
for i in range(3):
    eng.run(1.0, 5.0, 0.1, None, update=False)
    Y2 = eng.debug_buffer("Y").reshape(NT, V)
    print("repeat", i, O.norm_rel_err(Y2, ref), "bad rows", int((np.abs(Y2 - ref).max(axis=1) > 1e-3).sum()))
eng.close()
