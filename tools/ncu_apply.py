"""Apply-phase GEMM population for ncu (roofline evidence of the shipped GEMM).

Runs tn_hvp_environments at a config (untracked by the profiler), then ONE
tn_hvp_apply of `--batch` directions in sub-batches of `--max-batch` (bench.py's
launch configuration) inside cudaProfilerStart/Stop, with the library's GEMM
probe on: every DMMA GEMM launch of the apply is logged in launch order
(TN_GEMM_LOG: M N K batch opA opB ms A-batched B-batched has-beta), so the
n-th zgemm3m launch ncu captures (`--profile-from-start off -k regex:zgemm3m`)
is line n of the log.  Usage (on the GPU box):

  TN_GEMM_LOG=gpurun_out/apply_gemm_c4.log ncu --profile-from-start off \
     -k regex:zgemm3m --launch-skip S --launch-count C ... python tools/ncu_apply.py --config 4
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200 import _native as N  # noqa: E402
from paper_2604_20384_b200.api import SUB_BATCH, HVPEngine  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--max-batch", type=int, default=None)
a = ap.parse_args()
cfg = C.CONFIGS[a.config]
B = a.batch or SUB_BATCH[cfg.cid]
dev = torch.device("cuda")
ref = C.reference_mpo(cfg, device=dev)
K = C.num_gates(cfg.n, cfg.depth)
Gn = C.haar_gates(cfg.cid, K)
G = torch.tensor(Gn, device=dev)
V = torch.tensor(C.tangent_directions(cfg.cid, Gn, B), device=dev)
eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=a.max_batch or SUB_BATCH[cfg.cid])
eng.environments(G)
torch.cuda.synchronize()
N.tn_gemm_profile(1)
torch.cuda.profiler.start()
eng.apply(V)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ms, cmac = N.tn_gemm_profile(0)
print(f"apply {cfg.name} batch {B}: GEMM {ms:.1f} ms, {8 * cmac / ms / 1e9:.2f} TFLOP/s (algorithmic)")
