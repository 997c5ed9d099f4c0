"""Per-launch GEMM shapes and times of one apply (TN_GEMM_LOG), aggregated."""
import collections
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200 import _native as N  # noqa: E402
from paper_2604_20384_b200.api import HVPEngine  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cfg = C.CONFIGS[cid]
dev = torch.device("cuda")
ref = C.reference_mpo(cfg, device=dev)
K = C.num_gates(cfg.n, cfg.depth)
Gn = C.haar_gates(cfg.cid, K)
G = torch.tensor(Gn, device=dev)
V = torch.tensor(C.tangent_directions(cfg.cid, Gn, B), device=dev)
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=B)
eng.environments(G)
eng.apply(V)
torch.cuda.synchronize()
os.environ["TN_GEMM_LOG"] = "/tmp/gemm.log"
N.tn_gemm_profile(1)
eng.apply(V)
torch.cuda.synchronize()
ms, cm = N.tn_gemm_profile(0)
rows = [l.split() for l in open("/tmp/gemm.log")]
print(f"apply GEMMs: {len(rows)} launches, {ms:.1f} ms, {8*cm/ms/1e9:.2f} TF/s")
# bucket by work size
buck = collections.defaultdict(lambda: [0, 0.0, 0.0])
for M_, N_, K_, b, oa, ob, t in rows:
    w = int(M_) * int(N_) * int(K_) * int(b)
    key = f"{oa}{ob} 2^{max(0, w.bit_length()-1)}"
    buck[key][0] += 1
    buck[key][1] += float(t)
    buck[key][2] += w
for k, (n, t, w) in sorted(buck.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{k:12s} n={n:6d} {t:9.2f} ms  {8*w/t/1e9 if t else 0:6.2f} TF/s")
import math
def ctas(M_, N_, b):
    return math.ceil(int(M_) / 64) * math.ceil(int(N_) / 64) * int(b)
small = [r for r in rows if ctas(r[0], r[1], r[3]) < 148]
mid = [r for r in rows if 148 <= ctas(r[0], r[1], r[3]) < 592]
print("grids < 148 CTAs: n=%d  %.1f ms;  148..591: n=%d  %.1f ms" % (len(small), sum(float(r[6]) for r in small),
      len(mid), sum(float(r[6]) for r in mid)))
slow = sorted(rows, key=lambda r: -float(r[6]))[:15]
print("slowest launches (M N K batch op ms TF/s):")
for M_, N_, K_, b, oa, ob, t in slow:
    w = int(M_) * int(N_) * int(K_) * int(b)
    print(M_, N_, K_, b, oa + ob, t, f"{8*w/float(t)/1e9:.2f}")
