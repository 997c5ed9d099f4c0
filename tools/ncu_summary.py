"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`)
into per-kernel counts, summed duration and share.  Usage:
    python tools/ncu_summary.py launches.csv > profiles/<name>.md"""
import collections
import csv
import io
import sys

path = sys.argv[1]
with open(path) as f:
    text = f.read()
start = text.find('"ID"')
rows = list(csv.DictReader(io.StringIO(text[start:])))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    short = name.split("(")[0]
    if "zgemm3m_kernel" in name:
        short = "tn::zgemm3m_kernel (DMMA complex GEMM)"
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "nsecond")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
    agg[short][0] += 1
    agg[short][1] += v * scale
total = sum(t for _, t in agg.values())
n = sum(c for c, _ in agg.values())
print(f"# ncu launch list summary: {n} launches, {total:.1f} ms summed kernel time (cold-cache, serialised)")
print(f"# source: {path}\n")
print("| kernel | launches | ms | share |")
print("|---|---:|---:|---:|")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {c} | {t:.1f} | {t / total:.3f} |")
