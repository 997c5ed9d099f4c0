"""CPU checks of bench.py's contract pieces (no GPU): defaults, the bounded
oracle sample used for cpu_baseline / --impl reference."""
import sys

import bench
from tn_inputs import configs as C
from tn_inputs.reference import reference_mpo


def test_defaults(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert a.gpus == 1 and a.warmup >= 3 and a.steps >= 1 and a.config == 4 and a.impl == "ours"


def test_oracle_sample_is_bounded_and_positive():
    cfg = C.CONFIGS[2]
    ref = reference_mpo(C.reference_layers(cfg), cfg.n, cfg.chi)
    G = C.haar_gates(cfg.cid, C.num_gates(cfg.n, cfg.depth))
    rate, dt, done = bench.oracle_sample(cfg, [a.numpy() for a in ref], G, budget_s=2.0)
    assert rate > 0 and 0 < done <= cfg.n // 2 and dt < 30
