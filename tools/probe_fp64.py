"""FP64 roofline probes on the box: DMMA/DFMA loops (bin/fp64_peak), cuBLAS
ZGEMM via torch.matmul, our DMMA ZGEMM, cuSOLVER SVD timings.  One JSON line."""
import json
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import zgemm  # noqa: E402

out = {}
peak = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2604_20384_b200", "bin",
                    "fp64_peak")
out["loops"] = json.loads(subprocess.run([peak], capture_output=True, text=True).stdout)
dev = torch.device("cuda")


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


for n in (1024, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.complex128, device=dev)
    b = torch.randn(n, n, dtype=torch.complex128, device=dev)
    t = timeit(lambda: a @ b, 3 if n >= 8192 else 10)
    out[f"cublas_zgemm_{n}_tflops"] = 8 * n ** 3 / t / 1e12
    t = timeit(lambda: zgemm(a, b), 3 if n >= 8192 else 10)
    out[f"dmma_zgemm_{n}_tflops"] = 8 * n ** 3 / t / 1e12
    ad, bd = a.real.contiguous(), b.real.contiguous()
    t = timeit(lambda: ad @ bd, 3 if n >= 8192 else 10)
    out[f"cublas_dgemm_{n}_tflops"] = 2 * n ** 3 / t / 1e12
# shapes of the hot path at chi = 256: stacked (64*256 x 256) x (256 x 4096), batched 64 x (256 x 4096 x 256)
a = torch.randn(64 * 256, 256, dtype=torch.complex128, device=dev)
b = torch.randn(256, 4096, dtype=torch.complex128, device=dev)
t = timeit(lambda: zgemm(a, b))
out["dmma_stacked_16384x4096x256_tflops"] = 8 * 64 * 256 * 4096 * 256 / t / 1e12
a = torch.randn(1, 4096, 256, dtype=torch.complex128, device=dev)
b = torch.randn(64, 4096, 256, dtype=torch.complex128, device=dev)
t = timeit(lambda: zgemm(a, b, "C", "N"))
out["dmma_batched_CN_64x256x256x4096_tflops"] = 8 * 64 * 256 * 256 * 4096 / t / 1e12
for n in (256, 512, 1024):
    m = torch.randn(n, n, dtype=torch.complex128, device=dev)
    t = timeit(lambda: torch.linalg.svd(m, full_matrices=False), 3)
    out[f"torch_svd_{n}_ms"] = t * 1e3
print(json.dumps(out))
