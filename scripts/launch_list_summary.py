"""Summarise an ncu launch list (gpu__time_duration + DRAM bytes per launch) of
`bench.py --steps 2 --warmup 3` into one train step's kernel classes.

python scripts/launch_list_summary.py profiles/r02/ncu/launches_bench.csv > profiles/r02/ncu/launches_c3_step_summary.txt
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
L = collections.OrderedDict()
for d in data:
    L.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")),
                                                                           d["Metric Unit"])
launches = list(L.values())


def us(v):
    x, u = v
    return x / 1e3 if u in ("nsecond", "ns") else x * 1e3 if u == "msecond" else x


def mb(v):
    x, u = v
    return x / 1e6 if u == "byte" else x / 1e3 if u == "Kbyte" else x if u == "Mbyte" else x * 1e3


# a step starts at the set_scalars_kernel launch (graph replays keep the order)
starts = [i for i, l in enumerate(launches) if l["name"].startswith("set_scalars_kernel")]
if len(starts) < 2:
    starts = [i for i, l in enumerate(launches) if l["name"].startswith("void gather_rows_kernel")][0::2]
s0, s1 = starts[-3], starts[-2]  # the first timed step
step = launches[s0:s1]
tot = sum(us(l["gpu__time_duration.sum"]) for l in step)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for l in step:
    n = re.sub(r"\(.*", "", l["name"])
    a = agg[n]
    a[0] += 1
    a[1] += us(l["gpu__time_duration.sum"])
    a[2] += mb(l["dram__bytes_read.sum"])
    a[3] += mb(l["dram__bytes_write.sum"])
print("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv "
      "python bench.py --steps 2 --warmup 3 --no-cpu-baseline")
print(f"({sys.argv[1]}).  One train step (a timed step, CUDA-graph replay): {len(step)} launches, {tot / 1e3:.3f} ms "
      "serialised, cold-cache;")
print("every kernel of the step is listed, the recurrent scans included (under ncu they launch non-cooperatively);")
print("side-stream kernels (dropout masks, deferred dW columns, segments) run beside the scans in the timed step.")
print()
print(f"{'ms':>8s} {'share':>6s} {'n':>3s} {'avg us':>8s} {'DRAM rd MB':>10s} {'wr MB':>8s}  kernel")
for k, (n, t, r, w) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / 1e3:8.3f} {100 * t / tot:5.1f}% {n:3d} {t / n:8.1f} {r:10.1f} {w:8.1f}  {k[:100]}")
