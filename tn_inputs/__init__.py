"""Seeded synthetic inputs shared by the oracle and the CUDA path's tests.

Holds none of the method's arithmetic (no sweeps, environments, tangents,
projections): RNG streams, Haar gates, tangent directions built as G*S with S
skew-Hermitian, spin-chain Trotter circuits and the reference MPO they
compress to.
"""
from .configs import CONFIGS, Config, brickwall_sites, haar_gates, num_gates, small_case, tangent_directions  # noqa: F401
