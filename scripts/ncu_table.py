"""Compact table of the per-kernel ncu --set full captures (DIR/summary.txt from
scripts/ncu_summarize.py) and the dominant-kernel DRAM traffic for bench.py.

python scripts/ncu_table.py profiles/r02/ncu > profiles/r02/ncu/summary_table.txt
"""
import json
import os
import sys

d = sys.argv[1]
txt = open(os.path.join(d, "summary.txt")).read()
blocks = txt.split("== ")[1:]
print("ncu --set full --clock-control none --import-source on, one launch per kernel class of a c3 step "
      "(scripts/ncu_capture_all.sh, scripts/ncu_step.py); raw pages in *_raw.csv")
print(f"{'capture':14s} {'us':>8s} {'tensor%':>8s} {'dram%':>6s} {'DRAM rd MB':>10s} {'wr MB':>8s} {'L2%':>6s} "
      f"{'regs':>5s} {'grid':>5s}  kernel")
traffic = {}
for b in blocks:
    ls = b.splitlines()
    name = ls[0].split(":")[0]
    kern = ls[0].split(": ", 1)[1][:70] if ": " in ls[0] else ""
    m = {}
    for line in ls[1:]:
        p = line.split()
        if len(p) >= 2:
            m[p[0]] = (p[1], p[2] if len(p) > 2 else "")

    def val(k):
        v, u = m.get(k, ("0", ""))
        x = float(v.replace(",", ""))
        return x * 1e3 if u == "Gbyte" else x / 1e3 if u == "Kbyte" else x / 1e6 if u == "byte" else x

    def num(k):
        return float(m.get(k, ("0", ""))[0].replace(",", ""))
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    traffic[name] = round((rd + wr) * 1e6)
    print(f"{name:14s} {num('gpu__time_duration.sum'):8.1f} "
          f"{num('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'):8.1f} "
          f"{num('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} {rd:10.1f} {wr:8.1f} "
          f"{num('lts__throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
          f"{m.get('launch__registers_per_thread', ('?',))[0]:>5s} {m.get('launch__grid_size', ('?',))[0]:>5s}  {kern}")
dt = {"source": "ncu --set full, one launch each (scripts/ncu_capture_all.sh -> profiles/r02/ncu/*_raw.csv): "
                "dram__bytes_read.sum + dram__bytes_write.sum",
      "0": {"kernel": "logits GEMM gemm_tc_kernel<256,0,1,EpiStore,2,1>", "bytes_per_launch": traffic.get("logits_gemm")},
      "1": {"kernel": "lstm_bwd_multi<128,4> (scan pair)", "bytes_per_launch": traffic.get("bptt_pair")},
      "2": {"kernel": "lstm_fwd_tm<64> (scan pair)", "bytes_per_launch": traffic.get("fwd_pair")}}
json.dump(dt, open(os.path.join(os.path.dirname(os.path.normpath(d)), "..", "dominant_traffic.json"), "w"), indent=1)
