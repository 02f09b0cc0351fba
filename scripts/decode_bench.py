"""Translation throughput of the device beam search (decoding.py / cmt_beam_*):
beam 10, alpha 0.6, the c3 model (V=50000, E=H=1024, L=4, random init, so EOS
is rare and every search runs to its length cap 2*len+10), synthetic sources of
length 50, searched `batch` sentences at a time.

python scripts/decode_bench.py [bf16|fp32] [n_sentences] [batch]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_07170_b200 import decoding as D  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Model, ModelConfig, Rng  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "bf16"
nsent = int(sys.argv[2]) if len(sys.argv) > 2 else 128
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 128
cfg = ModelConfig(50000, 1024, 1024, 4, 0.2)
model = Model.new(cfg, Rng(1))
eng = Engine(cfg, mode=mode)
eng.upload(model.params)
g = np.random.default_rng(0)
srcs = [g.integers(4, 50000, size=50).tolist() for _ in range(nsent)]
dcfg = D.DecodeConfig(beam_size=10, length_penalty_alpha=0.6)
caps = [D.length_cap(dcfg, len(s)) for s in srcs]
D._run(eng, srcs[:min(batch, 8)], 10, 1, caps[:min(batch, 8)], 0.6)  # warm-up
t0 = time.perf_counter()
toks = 0
steps = 0
for c in range(0, nsent, batch):
    out = D._run(eng, srcs[c:c + batch], 10, 1, caps[c:c + batch], 0.6)
    toks += sum(len(t.tokens) + (0 if t.truncated else 1) for t in out)
    steps += max(caps[c:c + batch])
dt = time.perf_counter() - t0
print(json.dumps({"mode": mode, "model": "c3 (V=50000, E=H=1024, L=4), random init", "sentences": nsent,
                  "batch_sentences": batch, "src_len": 50, "beam": 10, "seconds": round(dt, 3),
                  "sentences_per_s": round(nsent / dt, 1), "output_tokens_per_s": round(toks / dt, 1),
                  "decoder_steps": steps, "ms_per_batched_step": round(1e3 * dt / steps, 3),
                  "rows_per_step": batch * 10}))
