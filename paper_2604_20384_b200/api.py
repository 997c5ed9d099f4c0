"""Thin torch-facing wrapper over the C ABI (device memory and streams only).

Every step of the computation runs in libtn_hvp.so; this module only
allocates torch tensors, passes their data pointers and the current stream.
"""
from __future__ import annotations

import torch

from . import _native as N

# Directions per tn_hvp_apply sub-batch at the five BASELINE.json configs (the
# launch configuration bench.py times and the full-size GPU tests use): the
# largest that keeps the tangent caches within HBM with the GEMM grids full.
SUB_BATCH = {1: 1, 2: 16, 3: 64, 4: 32, 5: 1}


def _require_cuda(t: torch.Tensor, name: str, dtype=torch.complex128):
    if not (t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise ValueError(f"{name}: expected a contiguous {dtype} CUDA tensor")


def _stream():
    return torch.cuda.current_stream().cuda_stream


class HVPEngine:
    """One context of the HVP kernel (n sites, depth D, bond cap chi).

    ref_sites: list of n complex128 tensors [b_s][4][b_{s+1}] holding
    U_ref/2^{n/2} (right-canonical, centre at site 0).
    """

    def __init__(self, n, depth, chi, ref_sites, first_offset=0, max_batch=64, device=None, flags=0, site_dim=4):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2604_20384_b200 needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.n, self.depth, self.chi, self.first_offset = n, depth, chi, first_offset
        self.K = N.tn_hvp_num_gates(n, depth, first_offset)
        self.ref_bonds = [1] + [int(a.shape[2]) for a in ref_sites]
        packed = torch.cat([a.to(self.device, torch.complex128).contiguous().reshape(-1) for a in ref_sites])
        self.site_dim = site_dim
        cfg = N.make_config(n, depth, chi, max_batch, first_offset, site_dim, N.TN_C128, self.device.index, flags)
        # the primal store is a caller-owned torch buffer (tn_hvp_query's size):
        # visible to torch's allocator and broadcastable in place (parallel.py)
        self.primal_bytes, self.workspace_bytes, self.per_direction_bytes = N.tn_hvp_query(cfg, self.ref_bonds)
        self.primal = torch.empty(max(self.primal_bytes, 256), dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            self.ctx = N.tn_hvp_setup(cfg, self.ref_bonds, packed.data_ptr(), _stream(), self.primal.data_ptr(),
                                      self.primal.numel())
        self.max_batch = max_batch
        self.scalars = torch.zeros(8, dtype=torch.float64, device=self.device)

    def close(self):
        if getattr(self, "ctx", None):
            torch.cuda.synchronize(self.device)
            N.tn_hvp_destroy(self.ctx)
            self.ctx = None
            self.primal = None

    def set_product_state(self, psi: torch.Tensor):
        """State mode: the bottom start |psi> = (x)_s psi[s] (psi [n, 2] complex128)."""
        _require_cuda(psi, "psi")
        N.tn_hvp_set_product_state(self.ctx, psi.data_ptr(), _stream())

    def set_reference(self, sites):
        """New reference / label tensors with the bonds given at construction."""
        packed = torch.cat([a.to(self.device, torch.complex128).contiguous().reshape(-1) for a in sites])
        N.tn_hvp_set_reference(self.ctx, packed.data_ptr(), _stream())
        torch.cuda.current_stream().synchronize()      # packed is a temporary

    def set_cache_budget(self, nbytes: int):
        """Cap on this context's per-point caches (0 = automatic)."""
        N.tn_hvp_set_cache_budget(self.ctx, nbytes)

    def trim_memory(self):
        """Drop per-point caches / graphs and return the library pool's unused memory."""
        N.tn_hvp_trim_memory(self.ctx, _stream())

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def environments(self, gates: torch.Tensor):
        """-> (scalars[8] device, grad_R [K,4,4] device). scalars = f, Re T, Im T, diag..."""
        _require_cuda(gates, "gates")
        gR = torch.empty(self.K, 4, 4, dtype=torch.complex128, device=self.device)
        N.tn_hvp_environments(self.ctx, gates.data_ptr(), self.scalars.data_ptr(), gR.data_ptr(), _stream())
        return self.scalars, gR

    def gradient_T(self):
        E = torch.empty(self.K, 4, 4, dtype=torch.complex128, device=self.device)
        N.tn_hvp_gradient_T(self.ctx, E.data_ptr(), _stream())
        return E

    def apply(self, dirs: torch.Tensor, aux: bool = False, out: torch.Tensor | None = None):
        """Riemannian HVPs for dirs [B,K,4,4] -> hess [B,K,4,4] (and (H_T, Omega) if aux)."""
        _require_cuda(dirs, "dirs")
        B = dirs.shape[0]
        hess = out if out is not None else torch.empty_like(dirs)
        ax = torch.empty(B * self.K * 16 + B, dtype=torch.complex128, device=self.device) if aux else None
        N.tn_hvp_apply(self.ctx, B, dirs.data_ptr(), hess.data_ptr(), ax.data_ptr() if aux else 0, _stream())
        if aux:
            return hess, ax[: B * self.K * 16].view(B, self.K, 4, 4), ax[B * self.K * 16:]
        return hess

    def step(self, gates: torch.Tensor, dirs: torch.Tensor, out: torch.Tensor | None = None):
        """environments(gates) + apply(dirs) in one fused call (tn_hvp_step):
        -> (scalars[8], grad_R [K,4,4], hess [B,K,4,4])."""
        _require_cuda(gates, "gates")
        _require_cuda(dirs, "dirs")
        gR = torch.empty(self.K, 4, 4, dtype=torch.complex128, device=self.device)
        hess = out if out is not None else torch.empty_like(dirs)
        N.tn_hvp_step(self.ctx, gates.data_ptr(), self.scalars.data_ptr(), gR.data_ptr(), dirs.shape[0],
                      dirs.data_ptr(), hess.data_ptr(), 0, _stream())
        return self.scalars, gR, hess

    def ti_environments(self, layer_gates: torch.Tensor):
        """Translation-invariant circuit (N2): layer gates [D,4,4] -> (scalars[8], grad_R [D,4,4])."""
        _require_cuda(layer_gates, "layer_gates")
        gR = torch.empty(self.depth, 4, 4, dtype=torch.complex128, device=self.device)
        N.tn_hvp_ti_environments(self.ctx, layer_gates.data_ptr(), self.scalars.data_ptr(), gR.data_ptr(), _stream())
        return self.scalars, gR

    def ti_apply(self, layer_dirs: torch.Tensor):
        """Riemannian HVPs on U(4)^D for layer-wise directions [B,D,4,4] -> [B,D,4,4]."""
        _require_cuda(layer_dirs, "layer_dirs")
        hess = torch.empty_like(layer_dirs)
        N.tn_hvp_ti_apply(self.ctx, layer_dirs.shape[0], layer_dirs.data_ptr(), hess.data_ptr(), _stream())
        return hess

    def cost(self, gates: torch.Tensor):
        _require_cuda(gates, "gates")
        sc = torch.zeros(8, dtype=torch.float64, device=self.device)
        N.tn_hvp_cost(self.ctx, gates.data_ptr(), sc.data_ptr(), _stream())
        return sc

    def primal_blob(self):
        return N.tn_hvp_primal_blob(self.ctx)

    def environments_part(self, gates: torch.Tensor, part: int):
        """Split primal: the bottom (0) or top (1) sweep only, into its store region."""
        _require_cuda(gates, "gates")
        N.tn_hvp_environments_part(self.ctx, gates.data_ptr(), part, _stream())

    def primal_region(self, part: int):
        """(byte offset, bytes) of side `part` inside the primal store."""
        return N.tn_hvp_primal_region(self.ctx, part)

    def environments_finish(self, gates: torch.Tensor):
        """Split primal: layer environments, E, f, grad_R once both regions are in place."""
        _require_cuda(gates, "gates")
        gR = torch.empty(self.K, 4, 4, dtype=torch.complex128, device=self.device)
        N.tn_hvp_environments_finish(self.ctx, gates.data_ptr(), self.scalars.data_ptr(), gR.data_ptr(), _stream())
        return self.scalars, gR

    def primal_store(self) -> torch.Tensor:
        """The primal store itself (uint8, tn_hvp_primal_blob's bytes; no copy)."""
        return self.primal[: self.primal_bytes]

    def invalidate_primal(self):
        """Before the store is overwritten by a collective: drop the old point."""
        st = self.primal_store()
        N.tn_hvp_primal_copy(self.ctx, st.data_ptr(), st.numel(), 1, _stream())

    def primal_imported(self, gates: torch.Tensor):
        _require_cuda(gates, "gates")
        N.tn_hvp_primal_imported(self.ctx, gates.data_ptr(), _stream())

    def split_stats(self):
        """Last primal pass: dict of QR-iteration fallbacks, deflation levels, noise-floor cuts,
        low-rank range-probe splits, rejected CholeskyQR2 moves and pair steps."""
        keys = ("qr_iteration_fallbacks", "deflation_levels", "noise_floor_cuts", "low_rank_splits",
                "cholqr_rejected", "pair_steps")
        return dict(zip(keys, N.tn_hvp_split_stats(self.ctx)))

    def work(self):
        """(complex MACs per direction of the last apply, complex MACs of the last primal pass)."""
        return N.tn_hvp_work(self.ctx)


def mpo_tebd(n: int, layers, chi: int, tol: float = 1e-14, device=None):
    """N4: the reference MPO U_ref/2^{n/2} of a gate sequence built on the GPU by
    tn_mpo_tebd.  layers: list of layers, each a list of (left site, 4x4 gate)
    applied in order (tn_inputs.models.trotter_layers).  -> list of n device
    tensors [b][4][b'] (right-canonical, centre at site 0, unit norm)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    sites = [int(i) for ly in layers for i, _ in ly]
    g = torch.tensor([[list(r) for r in gg] for ly in layers for _, gg in ly], dtype=torch.complex128,
                     device=dev) if sites else torch.zeros(1, 4, 4, dtype=torch.complex128, device=dev)
    cap = n * 16 * chi * chi
    out = torch.empty(cap, dtype=torch.complex128, device=dev)
    with torch.cuda.device(dev):
        bonds = N.tn_mpo_tebd(n, sites, g.data_ptr(), chi, tol, dev.index, out.data_ptr(), cap, _stream())
    res, o = [], 0
    for s in range(n):
        e = bonds[s] * 4 * bonds[s + 1]
        res.append(out[o:o + e].view(bonds[s], 4, bonds[s + 1]).clone())
        o += e
    return res


def riemannian_project(gates: torch.Tensor, Z: torch.Tensor) -> torch.Tensor:
    _require_cuda(gates, "gates")
    _require_cuda(Z, "Z")
    K = gates.shape[0]
    B = Z.numel() // (K * 16)
    out = torch.empty_like(Z)
    N.tn_riemannian_project(K, B, gates.data_ptr(), Z.data_ptr(), out.data_ptr(), _stream())
    return out


def zgemm(A: torch.Tensor, B: torch.Tensor, opa="N", opb="N", alpha=1.0, beta=0.0, C=None):
    """Batched DMMA complex GEMM on [batch, rows, cols] tensors (tests / probes)."""
    _require_cuda(A, "A")
    _require_cuda(B, "B")
    A3 = A if A.dim() == 3 else A[None]
    B3 = B if B.dim() == 3 else B[None]
    batch = max(A3.shape[0], B3.shape[0])
    M = A3.shape[1] if opa == "N" else A3.shape[2]
    K = A3.shape[2] if opa == "N" else A3.shape[1]
    Nn = B3.shape[2] if opb == "N" else B3.shape[1]
    if C is None:
        C = torch.zeros(batch, M, Nn, dtype=torch.complex128, device=A.device)
    sA = 0 if A3.shape[0] == 1 else A3.shape[1] * A3.shape[2]
    sB = 0 if B3.shape[0] == 1 else B3.shape[1] * B3.shape[2]
    N.tn_zgemm(opa, opb, M, Nn, K, complex(alpha), A3.data_ptr(), A3.shape[2], sA, B3.data_ptr(), B3.shape[2], sB,
               complex(beta), C.data_ptr(), Nn, M * Nn, batch, _stream())
    return C


def retract(gates: torch.Tensor, xi: torch.Tensor, alpha: float = 1.0) -> torch.Tensor:
    """Polar retraction R_G(alpha xi) = polar(G + alpha xi), gate-wise."""
    _require_cuda(gates, "gates")
    _require_cuda(xi, "xi")
    out = torch.empty_like(gates)
    N.tn_retract(gates.shape[0], gates.data_ptr(), xi.data_ptr(), float(alpha), out.data_ptr(), _stream())
    return out


def tangent_dot(A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    """Re <A_b, B_b> for [batch, ...] tangent vectors -> float64 [batch] (device)."""
    _require_cuda(A, "A")
    _require_cuda(B, "B")
    batch = A.shape[0] if A.dim() == 4 else 1
    n = A.numel() // batch
    out = torch.empty(batch, dtype=torch.float64, device=A.device)
    N.tn_tangent_dot(n, batch, A.data_ptr(), B.data_ptr(), out.data_ptr(), _stream())
    return out


def axpby(a, x: torch.Tensor, b, y: torch.Tensor) -> torch.Tensor:
    """y <- a x + b y in place (complex scalars a, b)."""
    _require_cuda(x, "x")
    _require_cuda(y, "y")
    N.tn_tangent_axpby(x.numel(), a, x.data_ptr(), b, y.data_ptr(), _stream())
    return y


def primal_export(eng: "HVPEngine") -> torch.Tensor:
    """The context's primal store (caller-owned uint8 tensor, tn_hvp_primal_blob's
    bytes); valid after environments / step.  No copy."""
    return eng.primal_store()


def primal_import(eng: "HVPEngine", buf: torch.Tensor, gates: torch.Tensor):
    """Fill the primal store from a buffer produced by primal_export at `gates`
    (same shapes) and mark it valid; a buffer that IS the store (in-place
    broadcast) is only marked.  TN_EINVAL if the store's point is not `gates`."""
    if buf.data_ptr() != eng.primal.data_ptr():
        N.tn_hvp_primal_copy(eng.ctx, buf.data_ptr(), buf.numel(), 1, _stream())
    eng.primal_imported(gates)


def pauli_basis(gates: torch.Tensor, first: int, count: int) -> torch.Tensor:
    """Pauli tangent basis vectors first..first+count-1 -> [count, K, 4, 4] (tn_pauli_basis)."""
    _require_cuda(gates, "gates")
    K = gates.shape[0]
    out = torch.empty((count, K, 4, 4), dtype=torch.complex128, device=gates.device)
    N.tn_pauli_basis(K, first, count, gates.data_ptr(), out.data_ptr(), _stream())
    return out


def pauli_coords(gates: torch.Tensor, X: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """<B_i, X_j> for every basis vector -> float64 [count, 16K] (tn_pauli_coords)."""
    _require_cuda(gates, "gates")
    _require_cuda(X, "X")
    K = gates.shape[0]
    X = X.reshape(-1, K, 4, 4)
    if out is None:
        out = torch.empty((X.shape[0], 16 * K), dtype=torch.float64, device=gates.device)
    N.tn_pauli_coords(K, X.shape[0], gates.data_ptr(), X.data_ptr(), out.data_ptr(), _stream())
    return out


def sym_eig(A: torch.Tensor, vectors: bool = False):
    """Eigenvalues (ascending) of the symmetric part of A (overwritten), the
    asymmetry (||A - A^T||_F, ||A||_F), and with vectors=True the eigenvectors
    as rows of A (tn_sym_eig)."""
    _require_cuda(A, "A", torch.float64)
    n = A.shape[0]
    w = torch.empty(n, dtype=torch.float64, device=A.device)
    asym = torch.empty(2, dtype=torch.float64, device=A.device)
    N.tn_sym_eig(n, A.data_ptr(), w.data_ptr(), asym.data_ptr(), vectors, _stream())
    return (w, asym, A) if vectors else (w, asym)
