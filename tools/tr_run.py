"""Config-5 style trust-region runs: independent problems sharded over ranks
(torchrun, NCCL), each rank optimising its problems sequentially with the GPU
HVP engine; final f values all-gathered to rank 0.  One JSON line per run."""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import HVPEngine  # noqa: E402
from paper_2604_20384_b200.parallel import shard  # noqa: E402
from paper_2604_20384_b200.trust_region import TRParams, TrustRegion  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--problems", type=int, default=None)
ap.add_argument("--outer", type=int, default=None)
ap.add_argument("--max-hvp", type=int, default=None)
ap.add_argument("--concurrent", type=int, default=1,
                help="problems in flight per GPU (one engine, stream and host thread each; memory permitting)")
a = ap.parse_args()
cfg = C.CONFIGS[a.config]
P = a.problems or cfg.extra.get("problems", 1)
outer = a.outer or cfg.extra.get("outer", 10)
max_hvp = a.max_hvp or cfg.extra.get("max_hvp", 20)
world = int(os.environ.get("WORLD_SIZE", 1))
rank = int(os.environ.get("RANK", 0))
if world > 1:
    import torch.distributed as dist
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("nccl")
dev = torch.device("cuda", torch.cuda.current_device())
t0 = time.time()
ref = C.reference_mpo(cfg, device=dev)
start, count = shard(P, rank, world)
mine = list(range(start, start + count))
lanes = max(1, min(a.concurrent, len(mine)))
engines = [HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=1) for _ in range(lanes)]
streams = [torch.cuda.Stream() for _ in range(lanes)]


def solve(p, lane):
    with torch.cuda.stream(streams[lane]):
        x0 = torch.tensor(C.trotter_init_gates(cfg, p), device=dev)
        tp = time.time()
        x, f, tr = TrustRegion(engines[lane], TRParams(outer=outer, max_hvp=max_hvp)).run(x0)
        torch.cuda.current_stream().synchronize()
    return {"problem": p, "f0": tr.records[0]["f"], "f": f, "hvps": tr.hvps, "grads": tr.grads,
            "seconds": time.time() - tp, "lane": lane,
            "trace": [{k: v for k, v in r.items() if k in ("iter", "f", "rho", "accepted", "n_hvp", "delta",
                                                             "tcg_stop")} for r in tr.records]}


results = []
if lanes == 1:
    results = [solve(p, 0) for p in mine]
else:   # problems are independent: interleave them over lanes (ctypes releases the GIL in the library)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=lanes) as ex:
        futs = []
        for i in range(0, len(mine), lanes):
            futs = [ex.submit(solve, p, j) for j, p in enumerate(mine[i:i + lanes])]
            results += [f.result() for f in futs]
if world > 1:
    fs = torch.zeros(P, dtype=torch.float64, device=dev)
    for r in results:
        fs[r["problem"]] = r["f"]
    dist.all_reduce(fs)           # disjoint problems: the sum is the gather
    gathered = fs.cpu().tolist()
else:
    gathered = [r["f"] for r in results]
if rank == 0:
    print(json.dumps({"config": cfg.name, "problems": P, "world": world, "outer": outer, "max_hvp": max_hvp,
                      "concurrent": lanes, "final_f": gathered, "rank0_runs": results,
                      "wall_s": time.time() - t0}))
if world > 1:
    dist.destroy_process_group()
