"""Repeated batch-1 tn_hvp_apply at one point (the truncated-CG pattern): wall
time of each call (1st eager, 2nd capture + replay, then replays), CUDA
events on the current stream.  Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20384_b200.api import HVPEngine  # noqa: E402
from tn_inputs import configs as C  # noqa: E402

out = {}
for cid in [int(x) for x in (sys.argv[1:] or ["3", "4"])]:
    cfg = C.CONFIGS[cid]
    dev = torch.device("cuda")
    ref = C.reference_mpo(cfg, device=dev)
    K = C.num_gates(cfg.n, cfg.depth)
    G = torch.tensor(C.haar_gates(cid, K), device=dev)
    V = torch.tensor(C.tangent_directions(cid, G.cpu().numpy(), 6), device=dev)
    eng = HVPEngine(cfg.n, cfg.depth, cfg.chi, ref, max_batch=1)
    eng.environments(G)
    st = torch.cuda.current_stream()
    ts, hs = [], []
    for i in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        hs.append(eng.apply(V[i:i + 1].contiguous()))
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    eng.close()
    out[cfg.name] = {"seconds_per_call": ts, "replay_speedup_vs_eager": ts[0] / min(ts[2:])}
    del ref
    torch.cuda.empty_cache()
print(json.dumps(out))
