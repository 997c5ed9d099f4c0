"""B200-native (sm_100a) Hessian-vector products for brickwall circuits vs an
MPO reference -- arXiv:2604.20384.  The compute path is libtn_hvp.so (C ABI in
include/tn_hvp.h); this package holds only the ctypes binding, a torch-facing
wrapper and the host-side drivers (batching/sharding, trust region)."""
from ._native import EXPORTS, LIB_PATH, TNError  # noqa: F401
