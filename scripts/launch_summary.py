"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import re
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for d in data:
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name, v, unit = d["Kernel Name"], float(d["Metric Value"].replace(",", "")), d["Metric Unit"]
    v = v / 1e3 if unit in ("nsecond", "ns") else v * 1e3 if unit == "msecond" else v
    short = re.sub(r"\(.*", "", name)[:90]
    m = re.match(r"void cmt::gemm_tc_kernel<(\d+), (\d+), (\d+), cmt::(\w+)>", name)
    if m:
        short = "tc<%s,%s,%s,%s>" % m.groups()
    m = re.match(r"void cmt::gemm_simt_kernel<cmt::(\w+), ([\w:]+)>", name)
    if m:
        short = "simt<%s,%s>" % m.groups()
    agg[short][0] += 1
    agg[short][1] += v
    tot += v
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}% n={n:5d} avg={t / n:9.1f}us  {k}")
print("total ms", tot / 1e3, "launches", sum(n for n, _ in agg.values()))
