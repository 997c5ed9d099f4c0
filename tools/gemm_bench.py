"""Time the DMMA complex GEMM (tn_zgemm) on the dominant C4 apply shapes
(tools/ncu_apply.py's GEMM log: the eight shapes carrying ~76% of the apply
flops) and report per-shape and flop-weighted algorithmic TFLOP/s (8 flop per
complex MAC).  Used to A/B kernel variants (environment switches are read at
library load, so run one process per variant).  One JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200 import _native as N  # noqa: E402

# (M, N, K, batch, opA, opB, A batched, B batched)
SHAPES = [(4096, 256, 256, 32, "N", "N", 1, 1), (32768, 1024, 256, 1, "N", "N", 0, 0),
          (1024, 1024, 256, 32, "N", "N", 1, 1), (256, 256, 4096, 32, "C", "N", 1, 1),
          (8192, 256, 4096, 1, "N", "C", 0, 0), (8192, 4096, 256, 1, "N", "N", 0, 0),
          (256, 1024, 1024, 32, "N", "N", 1, 0), (32768, 256, 1024, 1, "N", "C", 0, 0)]
dev = torch.device("cuda")
stream = torch.cuda.current_stream().cuda_stream
out = {"variant": os.environ.get("TN_GEMM_BSUM") and "bsum" or "default", "shapes": []}
tot_f = tot_t = 0.0
for M, Nn, K, B, oa, ob, ab, bb in SHAPES:
    a = torch.randn((B if ab else 1) * M * K, dtype=torch.complex128, device=dev)
    b = torch.randn((B if bb else 1) * K * Nn, dtype=torch.complex128, device=dev)
    c = torch.zeros(B * M * Nn, dtype=torch.complex128, device=dev)
    lda = K if oa == "N" else M
    ldb = Nn if ob == "N" else K

    def run():
        N.tn_zgemm(oa, ob, M, Nn, K, 1.0, a.data_ptr(), lda, M * K if ab else 0, b.data_ptr(), ldb,
                   K * Nn if bb else 0, 0.0, c.data_ptr(), Nn, M * Nn, B, stream)

    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    f = 8.0 * M * Nn * K * B
    tot_f += f
    tot_t += t
    out["shapes"].append({"shape": [M, Nn, K, B, oa + ob], "tflops": f / t / 1e12})
out["weighted_tflops"] = tot_f / tot_t / 1e12
print(json.dumps(out))
