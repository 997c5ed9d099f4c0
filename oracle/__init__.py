"""CPU oracle for the HVP kernel of arXiv:2604.20384 -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` leg may import or execute anything here.  The product path
(`paper_2604_20384_b200`) never imports it, and it never imports the product
path: the two share no code.  Everything is numpy complex128 (fp64).

Modules
  common  -- brickwall layout, Alg. 2 postprocessing in the
             X2 sign reading, Riemannian projections (App. E)
  dense   -- O1: exact dense Algorithm 1 on 2^n x 2^n
             operators, substitution HVP, finite differences;
             O2: the truncated definition on 4^n vectors
             with explicit Schmidt projectors
  mpo     -- O3: the same truncated definition realised with MPO sweeps
             (two-gauge channel tangent, App. D PAPER.md:976-1023 "fixed
             projectors"), generic layer environments for E_k and H_T
  trust   -- Riemannian trust region + truncated CG (Absil Alg. 10/11,
             PAPER.md:516) used to pin the driver

Parity status: every function is pinned in tests/test_oracle_*.py except the
truncated-regime VALUES at configs 2-5, which the paper does not print:
"parity unpinned" against the paper there (pinned only O3 == O2 structurally,
see DESIGN.md "Oracle pins").
"""
