"""A/B of engine options on the c3 step: device ms/step (CUDA events, graph
replay), alternating the two settings several times in one process.

python scripts/ab_option.py OPTION V0 V1 [reps] [steps]
python scripts/ab_option.py - "opt=v,opt2=v2" "opt=v,opt2=v2" [reps] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1802_07170_b200.engine import Engine  # noqa: E402
from paper_1802_07170_b200.model import Model, ModelConfig, Rng  # noqa: E402

opt = sys.argv[1]


def setting(x):
    if opt != "-":
        return ((opt, int(x)),)
    return tuple((kv.split("=")[0], int(kv.split("=")[1])) for kv in x.split(","))


v0, v1 = setting(sys.argv[2]), setting(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 20
V, E, H, L, B, S, T = bench.CONFIGS[os.environ.get("AB_CONFIG", "c3")]
cfg = ModelConfig(V, E, H, L, 0.2)
params = Model.new(cfg, Rng(1)).params
src, sm, tgt, tm = bench.synthetic_batch(V, S, T, B, seed=0)
fresh = os.environ.get("AB_FRESH") == "1"  # one engine per setting, options set before staging (e.g. bwd_bg)
engines = {}


def engine_for(v):
    if not fresh:
        if "one" not in engines:
            e = Engine(cfg, mode="bf16")
            e.upload(params)
            e.stage(src, sm, tgt, tm)
            engines["one"] = e
        e = engines["one"]
        for k_, x_ in v:
            e.set_option(k_, x_)
        return e
    if v not in engines:
        e = Engine(cfg, mode="bf16")
        for k_, x_ in v:
            e.set_option(k_, x_)
        e.upload(params)
        e.stage(src, sm, tgt, tm)
        engines[v] = e
    return engines[v]


rng = Rng(5)
res = {v0: [], v1: []}
for r in range(reps):
    for v in (v0, v1):
        eng = engine_for(v)
        for _ in range(3):
            eng.run(1.0, 5.0, 0.1, rng)
        eng.record(0)
        for _ in range(steps):
            eng.run(1.0, 5.0, 0.1, rng, asynchronous=True)
        eng.record(1)
        eng.wait()
        res[v].append(eng.elapsed_ms(0, 1) / steps)
for v in (v0, v1):
    print(f"{','.join(f'{k_}={x_}' for k_, x_ in v)}: " + " ".join(f"{x:.4f}" for x in res[v]) + f"  min {min(res[v]):.4f} ms/step", flush=True)
