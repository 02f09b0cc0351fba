"""Per-launch device timeline of one c3 train step (CUDA events after every
launch on the engine stream; no profiler).  python scripts/timeline.py [config]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Model, ModelConfig, Rng  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
opts = [a.split("=") for a in sys.argv[2:]]
V, E, H, L, B, S, T = bench.CONFIGS[name]
cfg = ModelConfig(V, E, H, L, 0.2)
model = Model.new(cfg, Rng(1))
eng = Engine(cfg, mode="bf16", device=0)
eng.upload(model.params)
for k, v in opts:
    eng.set_option(k, int(v))
src, sm, tgt, tm = bench.synthetic_batch(V, S, T, B, seed=0)
eng.stage(src, sm, tgt, tm)
rng = Rng(5)
for _ in range(3):
    eng.run(1.0, 5.0, 0.1, rng)
eng.set_option("timeline", 1)
eng.run(1.0, 5.0, 0.1, rng)
tl = eng.timeline()
eng.set_option("timeline", 0)
tot = sum(ms for _, ms in tl)
agg = collections.defaultdict(lambda: [0, 0.0])
for lab, ms in tl:
    key = lab.split(" t")[0] if lab.startswith("gemm") else lab
    agg[key][0] += 1
    agg[key][1] += ms
print(f"step total {tot:.3f} ms over {len(tl)} launches")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{ms:8.3f} ms {100 * ms / tot:5.1f}%  n={n:3d}  {k}")
print("\n# in order")
for lab, ms in tl:
    print(f"{ms * 1e3:9.1f} us  {lab}")
