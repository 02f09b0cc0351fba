"""Summarise ncu reports into small text/CSV files (run on the GPU box, where
the .ncu-rep files are too large to bring back).

python scripts/ncu_summarize.py DIR   -> DIR/<name>_raw.csv, DIR/summary.txt; removes the .ncu-rep files
"""
import csv
import glob
import io
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
]


def main(d):
    out = []
    for rep in sorted(glob.glob(os.path.join(d, "*.ncu-rep"))):
        name = os.path.basename(rep)[:-8]
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        with open(os.path.join(d, f"{name}_raw.csv"), "w") as f:
            f.write(raw)
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            out.append(f"== {name}: no data")
            continue
        hdr, units, vals = rows[0], rows[1], rows[2]
        get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        kname = get.get("Kernel Name", ("?", ""))[0]
        out.append(f"== {name}: {kname[:150]}")
        for k in KEYS:
            if k in get:
                out.append(f"   {k:70s} {get[k][0]:>20s} {get[k][1]}")
        for h in hdr:  # every tensor-pipe counter this ncu version exposes
            if "pipe_tensor" in h and "pct" in h:
                out.append(f"   {h:70s} {get[h][0]:>20s} {get[h][1]}")
        os.remove(rep)
    with open(os.path.join(d, "summary.txt"), "w") as f:
        f.write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncu")
