"""Summarise an ncu --set full capture of apply-phase zgemm3m launches
(tools/ncu_apply.py under `ncu --profile-from-start off -k regex:zgemm3m
--launch-skip S --launch-count C`), joined with the library's GEMM log of the
same run (line S + i = the i-th captured launch): per launch the shape, the
algorithmic DRAM bytes 16 (M K [x batch if A batched] + K N [x batch if B
batched] + M N batch [x2 with beta]), the measured dram__bytes_read+write, the
FP64-DMMA pipe utilisation and the algorithmic TFLOP/s (8 flop per complex
MAC).  Writes a markdown table (stdout) and, with --traffic, the JSON that
bench.py reads for roofline.traffic.

  python tools/ncu_gemm_summary.py raw.csv gemm.log --skip S [--traffic profiles/traffic_c4.json]
"""
import argparse
import csv
import io
import json

ap = argparse.ArgumentParser()
ap.add_argument("raw")
ap.add_argument("log")
ap.add_argument("--skip", type=int, required=True)
ap.add_argument("--traffic", default=None)
ap.add_argument("--source", default="")
a = ap.parse_args()

text = open(a.raw).read()
rows = list(csv.reader(io.StringIO(text[text.find('"ID"'):])))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
log = [ln.split() for ln in open(a.log) if ln.strip()]


def val(r, name, scale_units=True):
    v = r[col[name]].replace(",", "")
    if not v:
        return None
    x = float(v)
    if scale_units:
        u = units[col[name]]
        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
              "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(u, 1.0)
    return x


out = []
for i, r in enumerate(data):
    M, N, K, B, oa, ob, _, abat, bbat, beta = log[a.skip + i]
    M, N, K, B, abat, bbat, beta = int(M), int(N), int(K), int(B), int(abat), int(bbat), int(beta)
    alg = 16 * (M * K * (B if abat else 1) + K * N * (B if bbat else 1) + M * N * B * (2 if beta else 1))
    t = val(r, "gpu__time_duration.sum")
    dram = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    out.append({"M": M, "N": N, "K": K, "batch": B, "ops": oa + ob, "time_us": t * 1e6,
                "tflops": 8.0 * M * N * K * B / t / 1e12, "alg_bytes": alg, "dram_bytes": dram,
                "dram_over_alg": dram / alg,
                "dmma_pct": val(r, "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", False),
                "fp64_pct": val(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", False),
                "regs": val(r, "launch__registers_per_thread", False),
                "grid": val(r, "launch__grid_size", False)})
tt = sum(o["time_us"] for o in out)
print(f"# ncu --set full, {len(out)} consecutive apply-phase zgemm3m<78,78,2,2> launches (skip {a.skip}); "
      f"{a.source}")
print("# algorithmic bytes = 16 (M K + K N + M N) with batched operands counted per batch entry; "
      "TFLOP/s = 8 M N K batch / duration (ncu-serialised, cold cache)\n")
print("| M | N | K | batch | ops | us | TFLOP/s | DMMA pipe % | FP64 pipe % | alg MB | DRAM MB | DRAM/alg |")
print("|---:|---:|---:|---:|---|---:|---:|---:|---:|---:|---:|---:|")
for o in out:
    print(f"| {o['M']} | {o['N']} | {o['K']} | {o['batch']} | {o['ops']} | {o['time_us']:.0f} | {o['tflops']:.1f} | "
          f"{o['dmma_pct']:.1f} | {o['fp64_pct']:.1f} | {o['alg_bytes'] / 1e6:.2f} | {o['dram_bytes'] / 1e6:.2f} | "
          f"{o['dram_over_alg']:.2f} |")
w = {k: sum(o[k] * o["time_us"] for o in out) / tt for k in ("dmma_pct", "fp64_pct", "tflops")}
alg_mean = sum(o["alg_bytes"] for o in out) / len(out)
dram_mean = sum(o["dram_bytes"] for o in out) / len(out)
print(f"\ntime-weighted: DMMA pipe {w['dmma_pct']:.1f} %, FP64 pipe {w['fp64_pct']:.1f} %, "
      f"{w['tflops']:.1f} TFLOP/s algorithmic; mean per launch: algorithmic {alg_mean / 1e6:.2f} MB, "
      f"DRAM {dram_mean / 1e6:.2f} MB ({dram_mean / alg_mean:.2f}x)")
if a.traffic:
    json.dump({"dram_bytes_per_launch": dram_mean, "algorithmic_bytes_per_launch": alg_mean,
               "launches": len(out), "dmma_pipe_pct_time_weighted": w["dmma_pct"],
               "fp64_pipe_pct_time_weighted": w["fp64_pct"], "source": a.source,
               "population": "apply-phase zgemm3m launches (tools/ncu_apply.py), the kernel population of "
                             "bench.py's roofline.achieved"}, open(a.traffic, "w"), indent=1)
