"""Translation throughput on the engine: beam search (beam 10, alpha 0.6) and
greedy decoding of synthetic 50-token sources with the c3 model (random init,
so EOS is rare and every search runs to its length cap 2*50+10 = 110 steps).
python scripts/decode_bench.py [bf16|fp32] [n_sentences]"""
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
nsent = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = ModelConfig(50000, 1024, 1024, 4, 0.2)
model = Model.new(cfg, Rng(1))
eng = Engine(cfg, mode=mode)
eng.upload(model.params)
g = np.random.default_rng(0)
srcs = [g.integers(4, 50000, size=50).tolist() for _ in range(nsent + 1)]
dcfg = D.DecodeConfig(beam_size=10, length_penalty_alpha=0.6)
D.beam_search(srcs[0], model, dcfg, engine=eng)  # warm-up
steps = 0
orig = eng.decode_step


def counted(*a, **k):
    global steps
    steps += 1
    return orig(*a, **k)


eng.decode_step = counted
t0 = time.perf_counter()
toks = 0
for s in srcs[1:]:
    t = D.beam_search(s, model, dcfg, engine=eng)
    toks += len(t.tokens) + (0 if t.truncated else 1)
t_beam = time.perf_counter() - t0
beam_steps = steps
steps = 0
t0 = time.perf_counter()
for s in srcs[1:]:
    D.greedy_decode(s, model, 110, engine=eng)
t_greedy = time.perf_counter() - t0
print(json.dumps({"mode": mode, "model": "c3 (V=50000, E=H=1024, L=4), random init", "sentences": nsent,
                  "src_len": 50, "beam": 10,
                  "beam_search_s_per_sentence": t_beam / nsent, "beam_steps": beam_steps,
                  "beam_ms_per_step": 1e3 * t_beam / beam_steps, "beam_tokens_per_s": toks / t_beam,
                  "greedy_ms_per_step": 1e3 * t_greedy / steps, "greedy_steps": steps}))
