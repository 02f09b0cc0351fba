"""Benchmark: train target tokens/sec of one fwd+bwd+clipped-SGD step of the
CytonMT attention LSTM (BASELINE.json metric) on the paper-scale config
(configs[2]: 4-layer bi-encoder LSTM, emb/hidden 1024, vocab 50k, batch 128,
len 50) — the largest single-GPU config the metric is quoted on.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  ``value`` is device-timed with the batch
resident in HBM; ``e2e`` times the public API call (host ids/masks staged and
copied H2D, loss read back D2H) every step.  ``--impl reference`` times the
reference algorithm's CPU implementation (the numpy oracle port, the
reference itself being Python that cannot travel) on the host cores.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
import types

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (V, E, H, L, B, S, T)
    "c3": (50000, 1024, 1024, 4, 128, 50, 50),
    "c2": (30000, 512, 512, 2, 64, 50, 50),
    "tiny": (1000, 128, 128, 1, 16, 20, 20),
    "c5": (100000, 1024, 1024, 2, 256, 80, 80),
}
METRIC = "train target tokens/sec (fwd+bwd+update)"
CPU_SAMPLE_B = 16  # sentences per CPU-baseline step (bounded sample of the B=128 batch)
# the real reference (minmt.training.train_step) on the FULL c3 batch, measured
# in the survey container (8-core Xeon, numpy/OpenBLAS): BASELINE.md §2.2
REF_FULL = "163-180 tgt tok/s: minmt.train_step itself, full c3 batch (B=128, S=T=50), 8 cores, BASELINE.md 2.2"


def flops_per_step(V, E, H, L, B, S, T):
    """Algorithmic FLOPs: F_step = 3 F_fwd."""
    f = 8 * H * B * (2 * S * (E + H) + (L - 1) * S * 2 * H + T * (E + H) + (L - 1) * T * 2 * H)
    f += 6 * T * B * H * H + 4 * H * S * T * B + 2 * T * B * H * V
    return 3 * f


def synthetic_batch(V, S, T, B, seed):
    """ids uniform in [4, V), last target row EOS(3), masks all ones."""
    g = np.random.default_rng(seed)
    src = g.integers(4, V, (S, B)).astype(np.int64)
    tgt = g.integers(4, V, (T, B)).astype(np.int64)
    tgt[T - 1, :] = 3
    return src, np.ones((S, B), np.float32), tgt, np.ones((T, B), np.float32)


def peaks():
    """(burst bf16 TF/s, sustained bf16 TF/s, HBM GB/s, source) from MEASURED_PEAKS.json."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p["bf16_tflops_sustained"], p["hbm_gbs"], "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 1639.1, 1380.2, 6551.4, "fallback (SURVEY §8(d) / B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def mark(self):
        """Start of the timed region: samples before this point are dropped."""
        self.f.flush()
        try:
            with open(self.f.name) as fh:
                self.skip = sum(1 for _ in fh)
        except OSError:
            self.skip = 0

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        rows = rows[getattr(self, "skip", 0):]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for n, v in zip(names, r[2:]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(n)
            except (ValueError, IndexError):
                pass
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_oracle_rate(cfg_t, params, steps, warmup, sample_b=CPU_SAMPLE_B):
    """Reference algorithm on host cores (numpy oracle port) on a bounded sample."""
    from oracle import minmt_oracle as O
    V, E, H, L, B, S, T = cfg_t
    d = O.Dims(V, E, H, L, 0.2)
    names = [n for n, _ in O.registry(d)]
    src, sm, tgt, tm = synthetic_batch(V, S, T, sample_b, seed=0)
    gen = np.random.Generator(np.random.PCG64(5))
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        loss, g, _ = O.forward_backward(params, d, src, sm, tgt, tm, 0.1, gen=gen)
        O.sgd_step(params, g, names, 1.0, 5.0)
        del g
        if i >= warmup:
            times.append(time.perf_counter() - t0)
    ntok = float(tm.sum())
    return ntok / statistics.median(times), times


def step_breakdown(tl):
    """Group a per-launch timeline [(label, ms)] into kernel classes; keep the
    GEMM launches (label 'gemm MxNxK tile') for the GEMM-only roofline."""
    tot = sum(ms for _, ms in tl)
    cls = {"recurrent scans": 0.0, "tcgen05 GEMMs": 0.0, "CE + column sums": 0.0, "SGD + norm": 0.0,
           "attention core": 0.0, "dropout": 0.0, "dropout masks (beside the scans in the timed step)": 0.0,
           "other": 0.0}
    gemms = []
    for lab, ms in tl:
        if lab.startswith("gemm "):
            m, n, k = (int(x) for x in lab.split()[1].split("x"))
            gemms.append((m, n, k, ms))
            cls["tcgen05 GEMMs"] += ms
        elif lab.startswith("lstm"):
            cls["recurrent scans"] += ms
        elif lab.startswith(("ce_", "colsum", "sum_to")):
            cls["CE + column sums"] += ms
        elif lab.startswith(("sgd", "sumsq", "clip")):
            cls["SGD + norm"] += ms
        elif lab.startswith("attn"):
            cls["attention core"] += ms
        elif lab.startswith("dropout_mask"):
            cls["dropout masks (beside the scans in the timed step)"] += ms
        elif lab.startswith("dropout"):
            cls["dropout"] += ms
        else:
            cls["other"] += ms
    shares = {k: round(v / tot, 4) for k, v in cls.items()} if tot > 0 else {}
    shares["serialized_step_ms"] = round(tot, 4)
    return {"shares": shares, "gemms": gemms}


def gemm_roofline(bd, peak_tf):
    """GEMM-only fraction: sum of 2MNK over the step's tcgen05
    GEMM launches / their summed device time / the bf16 peak."""
    if not bd or not bd["gemms"]:
        return None
    fl = sum(2.0 * m * n * k for m, n, k, _ in bd["gemms"])
    ms = sum(x[3] for x in bd["gemms"])
    ach = fl / (ms / 1e3) / 1e12
    return {"achieved": ach, "peak": peak_tf, "unit": "TFLOP/s", "frac": ach / peak_tf, "launches": len(bd["gemms"]),
            "flops_per_step": fl, "ms_per_step": ms,
            "source": "per-launch CUDA events on the engine stream (one untimed step, side stream off)"}


def hbm_classes(tl, cfg_t, peak_hbm):
    """Achieved HBM bandwidth of the bandwidth-bound kernel classes of one
    serialised step (algorithmic bytes) against the HBM peak."""
    V, E, H, L, B, S, T = cfg_t
    NS, NT = S * B, T * B
    # dense (non-embedding) parameters: 3 layers read E + H inputs, 2(L-1) read 2H; attention; output
    dense = 3 * ((E + H) * 4 * H + 4 * H) + 2 * (L - 1) * (2 * H * 4 * H + 4 * H) + 3 * H * H + H * V + V
    cls = {
        # two-pass CE: stats read the bf16 logits, the gradient pass reads and rewrites them
        "CE (ce_stats + ce_grad)": (("ce_stats", "ce_grad"), 3 * 2.0 * NT * V),
        # norm (fp32 grad read) + SGD (fp32 w, g read, w write, bf16 shadow write), dense part only
        "norm + SGD (dense)": (("sumsq", "sgd_dense", "clip"), (4 + 14) * float(dense)),
        # dropout sites with their masks generated ahead (dropout_mask_kernel beside the
        # recurrent scans): read x (bf16; enc.l2's site x and x2; H_o's fp32) and the keep
        # byte, write y (bf16)
        "dropout apply (7 sites)": (("dropout_apply",),
                                    float(H) * (NS * (7 + 5 * (L - 2)) + NT * 5 * (L - 1) + NT * 7)),
        # fused draw-and-apply (fp32 mode / schedules without the side stream): x, y, keep
        "dropout fused (7 sites)": (("dropout_fwd",), 5.0 * H * ((L - 1) * NS + (L - 1) * NT + NT)),
    }
    out = {}
    for name, (prefixes, nbytes) in cls.items():
        ms = sum(m for lab, m in tl if lab.startswith(prefixes))
        if ms > 0:
            gbs = nbytes / (ms / 1e3) / 1e9
            out[name] = {"bytes": nbytes, "ms": round(ms, 4), "GB/s": round(gbs, 1), "frac": round(gbs / peak_hbm, 3)}
    return out


def run_reference(args, cfg_t):
    """--impl reference: the reference's CPU implementation of the path, timed here."""
    from paper_1802_07170_b200.model import Model, ModelConfig, Rng
    V, E, H, L, B, S, T = cfg_t
    model = Model.new(ModelConfig(V, E, H, L, 0.2), Rng(1))
    params = {b.name: b.var.data for b in model.params.blocks()}
    rate, times = cpu_oracle_rate(cfg_t, params, args.steps, args.warmup)
    cores = os.cpu_count()
    sample = f"{CPU_SAMPLE_B} of {B} sentences (S=T={S}) per step, {args.steps} steps after {args.warmup} warm-up"
    out = {
        "metric": METRIC, "value": rate, "unit": "tgt_tok/s", "n_gpus": args.gpus, "steps": args.steps,
        # the measured step of the sample (what the timed loop ran); the full
        # c3 batch would take B / sample times longer
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
        "ms_per_step_full_batch_est": 1e3 * statistics.median(times) * B / CPU_SAMPLE_B,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": args.config, "vocab": V, "emb": E, "hidden": H, "depth": L, "batch": B,
                   "src_len": S, "tgt_len": T},
        "cpu_baseline": {"value": rate, "unit": "tgt_tok/s", "cores": cores, "kind": "port", "sample": sample,
                         "reference_full_batch": REF_FULL},
        "e2e": {"value": rate, "unit": "tgt_tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=list(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg_t = CONFIGS[args.config]
    V, E, H, L, B, S, T = cfg_t

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, cfg_t)
        return

    import torch
    from paper_1802_07170_b200.engine import Engine, launch_count
    from paper_1802_07170_b200.model import Batch, Model, ModelConfig, Rng

    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    cfg = ModelConfig(V, E, H, L, 0.2)
    model = Model.new(cfg, Rng(1))
    eng = Engine(cfg, mode="bf16", device=local)
    for kv in filter(None, os.environ.get("CMT_OPTIONS", "").split(",")):  # experiments: k=v engine options
        k, v = kv.split("=")
        eng.set_option(k.strip(), int(v))
    eng.upload(model.params)
    if world > 1:
        eng.set_dp(dist, rank, world)
    src, sm, tgt, tm = synthetic_batch(V, S, T, B, seed=rank)
    batch = Batch(src, tgt, sm, tm)
    rng = Rng(5 + rank)
    from paper_1802_07170_b200 import dp as dpmod
    ntok_local = float(tm.sum())
    ntok_global = dpmod.global_ntok(tm, dist)
    lr, clip, eps = 1.0, 5.0, 0.1

    eng.stage(src, sm, tgt, tm)
    if dist:  # the ranks agree on the embedding rows the step exchanges (dp.exchange_rows)
        dpmod.exchange_rows(eng, dist)
    # the warm-up steps capture the step graph that the timed steps replay (the
    # engine captures a shape's second step; data parallel steps stay eager)
    for _ in range(args.warmup):
        eng.run(lr, clip, eps, rng, global_ntok=ntok_global)

    # ---- device-resident timing ----
    if dist:
        dist.barrier()
    torch.cuda.synchronize(local)
    clocks = ClockSampler(local)
    time.sleep(0.5)  # let nvidia-smi start sampling before the timed region
    clocks.mark()
    l0 = launch_count()
    g0 = eng.stat("graph_replays")[0]
    eng.record(0)
    for _ in range(args.steps):
        eng.run(lr, clip, eps, rng, global_ntok=ntok_global, asynchronous=True)
    eng.record(1)
    r = eng.wait()
    ms_total = eng.elapsed_ms(0, 1)
    launches = (launch_count() - l0) // args.steps
    graph_replays = int(eng.stat("graph_replays")[0] - g0)
    ck = clocks.stop()

    # ---- kernel-class probes: the same K steps again, launched eagerly with
    # CUDA events bracketing the logits GEMM, BPTT-scan and forward-scan launches
    # on the engine stream (event-record nodes inside the captured graph add
    # ~0.3 ms to a step, so the headline pass above runs without them) ----
    eng.set_option("graph", 0)
    eng.set_option("time_dominant", 7)
    eng.run(lr, clip, eps, rng, global_ntok=ntok_global)
    for c in (0, 1, 2):
        eng.stat(f"probe_ms:{c}")  # drop the warm-up step's probes
    eng.record(4)
    for _ in range(args.steps):
        eng.run(lr, clip, eps, rng, global_ntok=ntok_global, asynchronous=True)
    eng.record(5)
    eng.wait()
    ms_probe_pass = eng.elapsed_ms(4, 5) / args.steps
    probes = {c: eng.stat(f"probe_ms:{c}") for c in (0, 1, 2)}  # (mean ms per launch, launches)
    eng.set_option("time_dominant", 0)
    eng.set_option("graph", 1)

    # ---- per-launch breakdown of one (untimed) step: CUDA events after every
    # launch on the engine stream (the side-stream overlap is off in this mode) ----
    breakdown = None
    if rank == 0:
        eng.set_option("timeline", 1)
        eng.run(lr, clip, eps, rng, global_ntok=ntok_global)
        tl = eng.timeline()
        eng.set_option("timeline", 0)
        breakdown = step_breakdown(tl)

    # ---- end-to-end through the public API (host buffers, H2D + D2H inside) ----
    # The reference-facing call: training.train_step(model, batch, cfg, lr, rng)
    # (training.py:145-159) with device-resident parameters (sync="lazy", the
    # mode install() wires into the reference Trainer): every step validates and
    # converts the host ids/masks, segment-sorts the embedding rows, copies them
    # H2D, runs the step and reads the loss back as a Python float.
    from paper_1802_07170_b200 import training as TR
    TR._ENGINES[model] = eng
    tcfg = types.SimpleNamespace(grad_clip_norm=clip, label_smoothing=eps)
    if dist is None:  # warm-up of the API path (its first steps capture the step graph)
        for _ in range(2):
            TR.train_step(model, batch, tcfg, lr, rng, sync="lazy")
    if dist:
        dist.barrier()
    eng.record(2)
    t0 = time.perf_counter()
    if dist is None:
        for _ in range(args.steps):
            loss = TR.train_step(model, batch, tcfg, lr, rng, sync="lazy")
        e2e_api = "paper_1802_07170_b200.training.train_step (reference signature, sync='lazy')"
    else:  # data parallel: the step needs the global token count (dp.global_ntok), which the
        # reference signature does not carry -> the engine's public training loop
        for loss, _ in eng.pipeline((batch for _ in range(args.steps)), lr, clip, eps, rng,
                                    global_ntok=ntok_global):
            pass
        e2e_api = "Engine.pipeline (data parallel: global token count per step)"
    t_e2e = time.perf_counter() - t0
    eng.record(3)
    ms_e2e = max(1e3 * t_e2e, eng.elapsed_ms(2, 3))
    # Engine.pipeline: the same per-step work with batch i+1 staged on the host
    # while step i runs on the device
    t0 = time.perf_counter()
    for _ in eng.pipeline((batch for _ in range(args.steps)), lr, clip, eps, rng, global_ntok=ntok_global):
        pass
    ms_pipe = 1e3 * (time.perf_counter() - t0)

    ms_step = ms_total / args.steps
    if dist:
        t = torch.tensor([ms_step, ms_e2e / args.steps], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step, ms_e2e_step = t.tolist()
    else:
        ms_e2e_step = ms_e2e / args.steps
    value = world * ntok_local / (ms_step / 1e3)
    e2e_value = world * ntok_local / (ms_e2e_step / 1e3)
    pipe_value = world * ntok_local / (ms_pipe / args.steps / 1e3)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    burst_tf, sus_tf, peak_hbm, peak_src = peaks()
    # the run's clocks decide the denominator: burst unless the power cap engaged
    capped = bool(ck and "sw_power_cap" in ck.get("reasons", []))
    peak_tf = sus_tf if capped else burst_tf
    peak_src += ", sustained bf16 (power cap seen)" if capped else ", burst bf16 (no power cap in the timed region)"
    # roofline of the kernel class with the largest device time per step
    # (CUDA events around its launches on the engine stream, inside the timed steps)
    rec = 2.0 * B * 4 * H * H * (L * T + (L + 1) * S)  # recurrent products of all 2L+1 scans
    kinds = {
        0: ("logits GEMM tanh(W_o^T H_o + b_o) (tcgen05 CTA-pair, gemm_tc_kernel)", 2.0 * T * B * H * V),
        1: ("recurrent BPTT scans (lstm_bwd_multi, persistent tcgen05)", rec),
        2: ("recurrent forward scans (lstm_fwd_tm / lstm_fwd_multi, persistent tcgen05)", rec),
    }
    classes = {}
    for c, (name, fl) in kinds.items():
        mean_ms, n = probes[c]
        ms = mean_ms * n / args.steps
        if ms > 0:
            ach = fl / (ms / 1e3) / 1e12
            classes[c] = {"kernel": name, "ms_per_step": ms, "launches_per_step": n / args.steps,
                          "flops_per_step": fl, "achieved": ach, "frac": ach / peak_tf}
    dom = max(classes, key=lambda c: classes[c]["ms_per_step"]) if classes else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "dominant_traffic.json")
    if os.path.exists(tpath) and dom is not None:
        try:
            tj = json.load(open(tpath))
            traffic = tj.get(str(dom), {}).get("bytes_per_launch") if isinstance(tj.get(str(dom)), dict) else None
        except Exception:
            traffic = None
    fstep = flops_per_step(*cfg_t)
    # per step: int32 source ids, shifted and gold target ids, fp32 masks; the
    # embedding segments are sorted on the device (host-built and copied only
    # in data-parallel steps)
    h2d = S * B * 4 + 2 * T * B * 4 + S * B * 4 + T * B * 4
    if dist:
        h2d += 4 * (3 * (S + T) * B + 2)
    out = {
        "metric": METRIC, "value": value, "unit": "tgt_tok/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded ids, random-init weights)",
        "config": {"workload": args.config, "vocab": V, "emb": E, "hidden": H, "depth": L, "batch_per_gpu": B,
                   "global_batch": B * world, "src_len": S, "tgt_len": T, "dropout": 0.2, "label_smoothing": eps,
                   "clip": clip, "parallelism": f"dp{world}",
                   "l2": f"working set > L2 (bf16 logits alone {T * B * V * 2 / 1e9:.2f} GB per step)"},
        "e2e": {"value": e2e_value, "unit": "tgt_tok/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 40,
                "api": e2e_api},
        "e2e_pipeline": {"value": pipe_value, "unit": "tgt_tok/s",
                         "api": "Engine.pipeline (host staging of batch i+1 overlaps step i)"},
        "gpu_launches": int(launches),
        "cuda_graph": {"replays_in_timed_steps": graph_replays, "steps": args.steps,
                       "note": "each timed step replays the step graph captured in the warm-up "
                               "(gpu_launches counts the kernel nodes of the replayed graph)"},
        "probe_pass": {"ms_per_step": ms_probe_pass, "launch": "eager",
                       "note": "roofline / roofline_classes: CUDA events around the class's launches on the "
                               "engine stream over K further steps of the same workload"},
        "roofline": None if dom is None else {
            "bound": "tensor", "kernel": classes[dom]["kernel"], "achieved": classes[dom]["achieved"],
            "peak": peak_tf, "unit": "TFLOP/s", "frac": classes[dom]["frac"], "traffic": traffic,
            "flops_per_launch": classes[dom]["flops_per_step"] / classes[dom]["launches_per_step"],
            "launch_ms": classes[dom]["ms_per_step"] / classes[dom]["launches_per_step"],
            "launches_per_step": classes[dom]["launches_per_step"], "peak_source": peak_src},
        "roofline_classes": {v["kernel"].split(" (")[0]: {k: (round(x, 4) if isinstance(x, float) else x)
                                                       for k, x in v.items() if k != "kernel"}
                             for v in classes.values()},
        "hbm_classes": hbm_classes(tl, cfg_t, peak_hbm) if breakdown else None,
        "gemm_roofline": gemm_roofline(breakdown, peak_tf),
        "breakdown": breakdown and breakdown["shares"],
        "step_roofline": {"flops_per_step": fstep, "achieved_tflops": fstep / (ms_step / 1e3) / 1e12,
                          "frac": fstep / (ms_step / 1e3) / 1e12 / peak_tf},
        "src_tok_per_s": world * float(sm.sum()) / (ms_step / 1e3),
        "loss_last": loss,
        "clocks": ck,
    }
    if world == 1 and not args.no_cpu_baseline:
        params = {b.name: b.var.data for b in model.params.blocks()}
        rate, times = cpu_oracle_rate(cfg_t, params, 2, 0)
        out["cpu_baseline"] = {"value": rate, "unit": "tgt_tok/s", "cores": os.cpu_count(), "kind": "port",
                               "sample": f"numpy oracle, {CPU_SAMPLE_B} of {B} sentences (S=T={S}), "
                                         f"median of 2 steps ({sum(times):.1f} s)",
                               "reference_full_batch": REF_FULL if args.config == "c3" else None}
    print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
