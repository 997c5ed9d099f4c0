"""Summarise an ncu --set full raw CSV of the memory-bound kernels (gate application, environment extraction):
per launch the duration, DRAM bytes read + written, achieved DRAM GB/s and its share of the measured HBM peak.
    python tools/ncu_hbm_summary.py raw.csv [peak_gbs] > profiles/<name>.md"""
import csv
import io
import json
import os
import sys

path = sys.argv[1]
peak = float(sys.argv[2]) if len(sys.argv) > 2 else None
if peak is None:
    mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    peak = json.load(open(mp))["hbm_gbs"] if os.path.exists(mp) else 6525.6
text = open(path).read()
start = text.find('"ID"')
rows = list(csv.reader(io.StringIO(text[start:])))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def val(r, name):
    v = r[col[name]].replace(",", "")
    return float(v) if v not in ("", "n/a") else float("nan")


def scaled(r, name, table):
    return val(r, name) * table.get(units[col[name]], 1.0)


BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TIME = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
print(f"| kernel | grid | us | DRAM read MB | DRAM write MB | GB/s | of {peak:.0f} GB/s | L2 hit % |")
print("|---|---:|---:|---:|---:|---:|---:|---:|")
tot_b = tot_t = 0.0
for r in data:
    if len(r) < len(hdr):
        continue
    name = r[col["Kernel Name"]].split("(")[0]
    t = scaled(r, "gpu__time_duration.sum", TIME)
    rd = scaled(r, "dram__bytes_read.sum", BYTES)
    wr = scaled(r, "dram__bytes_write.sum", BYTES)
    l2 = val(r, "lts__t_sector_hit_rate.pct") if "lts__t_sector_hit_rate.pct" in col else float("nan")
    gbs = (rd + wr) / t / 1e9
    tot_b += rd + wr
    tot_t += t
    print(f"| `{name}` | {r[col['Grid Size']]} | {t * 1e6:.1f} | {rd / 1e6:.2f} | {wr / 1e6:.2f} | {gbs:.0f} | {gbs / peak:.2f} | {l2:.0f} |")
if tot_t:
    print(f"\ntime-weighted: {tot_b / tot_t / 1e9:.0f} GB/s = {tot_b / tot_t / 1e9 / peak:.2f} of the measured HBM peak {peak:.0f} GB/s")
