"""Dense primitives of the reference (`densela.py:79-217`) on the GPU.

`cholesky`, `tri_solve`, `pivoted_qr` and `matmul` keep the reference's
names, arguments, return types (`CholeskyFactor`, `PivotedQR`), error
behaviour (ValueError for NaN/Inf or asymmetric input, NotSPDError on a
pivot below 1e-14 x the largest diagonal entry, ShapeMismatchError) and the
analytic flop tally `FLOPS`.  The arithmetic runs in the native library's
per-primitive entry points (`sgf_potrf_batched`, `sgf_trsm_batched`,
`sgf_qrcp_batched`, `sgf_gemm`, include/sgf.h); the `*_batched` variants take
lists of matrices and make one call for all of them.  Host arrays are copied
to the device through torch buffers (plumbing only) and results copied back.

These are the building blocks the factorization uses, exposed one call at a
time for callers and for the reference's own primitive tests
(tests/test_densela_gpu.py); `factorize` itself runs its batched level
kernels directly.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import NotSPDError, ShapeMismatchError

CHOL_PIVOT_RTOL = 1e-14
DEFAULT_RANK_TOL = 1e-10


class FlopCounter(object):
    """Running tally of analytic flop counts (reference densela.py:24-40)."""

    def __init__(self):
        self.total = 0

    def add(self, flops):
        self.total += int(flops)

    def reset(self):
        self.total = 0


FLOPS = FlopCounter()


@dataclass
class CholeskyFactor:
    """Lower-triangular factor L with A = L L^T."""

    L: np.ndarray

    @property
    def size(self):
        return self.L.shape[0]


@dataclass
class PivotedQR:
    """A[:, perm] = Q R (reference densela.py:61-76)."""

    Q: np.ndarray
    R: np.ndarray
    perm: np.ndarray
    rank: int


def _as_matrix(a):
    """reference densela.py:43-49 (the NaN/Inf check itself runs on the device
    in cholesky; pivoted_qr keeps the host check of the reference)."""
    a = np.asarray(a, dtype=float)
    if a.ndim != 2:
        raise ShapeMismatchError(f"expected a 2-d array, got shape {a.shape}")
    return a


def _dev(device=0):
    import torch

    return torch, N.context(device), torch.device("cuda", device)


def _arr(vals, ctype):
    return (ctype * max(len(vals), 1))(*vals)


def cholesky_batched(mats, device=0):
    """Cholesky of every matrix in `mats` in one native call."""
    torch, ctx, dev = _dev(device)
    A = [_as_matrix(a) for a in mats]
    for a in A:
        if a.shape[0] != a.shape[1]:
            raise ShapeMismatchError(f"cholesky needs a square matrix, got {a.shape}")
    dA = [torch.as_tensor(np.ascontiguousarray(a), device=dev) for a in A]
    dL = [torch.empty_like(t) for t in dA]
    b = len(A)
    m = _arr([a.shape[0] for a in A], C.c_int32)
    status = (C.c_int32 * max(b, 1))()
    pidx = (C.c_int32 * max(b, 1))()
    pval = (C.c_double * max(b, 1))()
    N.order_after_torch(ctx, device)
    st = N.lib().sgf_potrf_batched(ctx, b, m, _arr([t.data_ptr() for t in dA], C.c_void_p), m,
                                   _arr([t.data_ptr() for t in dL], C.c_void_p), m, status, pidx, pval)
    N.raise_for(st, ctx)
    out = []
    for i, a in enumerate(A):
        if status[i] == N.SGF_INVALID_ARG:
            raise ValueError("matrix contains NaN or Inf entries")
        if status[i] == N.SGF_NON_SYMMETRIC:
            asym = np.abs(a - a.T).max()
            raise ValueError(f"matrix is not symmetric (asymmetry {asym:.2e})")
        if status[i] == N.SGF_NOT_SPD:
            raise NotSPDError(f"non-positive pivot {pval[i]:.3e} at index {pidx[i]}")
        FLOPS.add(a.shape[0] ** 3 // 3)
        out.append(CholeskyFactor(dL[i].cpu().numpy()))
    return out


def cholesky(A, device=0):
    """Cholesky factorization of a dense SPD matrix (reference densela.py:87-116)."""
    return cholesky_batched([A], device)[0]


_MODES = {"left": 0, "left_t": 1, "right_t": 2}


def tri_solve(chol, B, mode="left", device=0):
    """L^{-1} B ("left"), L^{-T} B ("left_t") or B L^{-T} ("right_t")
    (reference densela.py:119-146)."""
    torch, ctx, dev = _dev(device)
    L = chol.L if isinstance(chol, CholeskyFactor) else np.asarray(chol, dtype=float)
    B = np.asarray(B, dtype=float)
    vec = B.ndim == 1
    if vec:
        B = B[:, None]
    m = L.shape[0]
    if mode not in _MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if mode in ("left", "left_t"):
        if B.shape[0] != m:
            raise ShapeMismatchError(f"solve: L is {L.shape}, B is {B.shape}")
        nrhs = B.shape[1]
    else:
        if B.shape[1] != m:
            raise ShapeMismatchError(f"solve: L is {L.shape}, B is {B.shape}")
        nrhs = B.shape[0]
    FLOPS.add(m * m * nrhs)
    dL = torch.as_tensor(np.ascontiguousarray(L), device=dev)
    dB = torch.as_tensor(np.ascontiguousarray(B), device=dev)
    dX = torch.empty_like(dB)
    N.order_after_torch(ctx, device)
    st = N.lib().sgf_trsm_batched(ctx, 1, _arr([m], C.c_int32), _arr([nrhs], C.c_int32),
                                  _arr([_MODES[mode]], C.c_int32), _arr([dL.data_ptr()], C.c_void_p),
                                  _arr([dL.shape[1]], C.c_int32), _arr([dB.data_ptr()], C.c_void_p),
                                  _arr([dB.shape[1]], C.c_int32), _arr([dX.data_ptr()], C.c_void_p),
                                  _arr([dX.shape[1]], C.c_int32))
    N.raise_for(st, ctx)
    X = dX.cpu().numpy()
    return X[:, 0] if vec else X


def pivoted_qr_batched(mats, rank_tol=DEFAULT_RANK_TOL, full_q=False, device=0):
    """pivoted_qr of every matrix in `mats` in one native call."""
    torch, ctx, dev = _dev(device)
    A = [_as_matrix(a) for a in mats]
    for a in A:
        if not np.isfinite(a).all():
            raise ValueError("matrix contains NaN or Inf entries")
    b = len(A)
    dA, dQ, dR, dP = [], [], [], []
    for a in A:
        m, c = a.shape
        kmax = min(m, c)
        dA.append(torch.as_tensor(np.ascontiguousarray(a) if a.size else np.zeros((max(m, 1), max(c, 1))),
                                  device=dev))
        dQ.append(torch.empty((max(m, 1), max(m if full_q else kmax, 1)), dtype=torch.float64, device=dev))
        dR.append(torch.empty((max(kmax, 1), max(c, 1)), dtype=torch.float64, device=dev))
        dP.append(torch.empty(max(c, 1), dtype=torch.int32, device=dev))
    rank = (C.c_int32 * max(b, 1))()
    steps = (C.c_int32 * max(b, 1))()
    N.order_after_torch(ctx, device)
    st = N.lib().sgf_qrcp_batched(ctx, b, _arr([a.shape[0] for a in A], C.c_int32),
                                  _arr([a.shape[1] for a in A], C.c_int32), _arr([t.data_ptr() for t in dA], C.c_void_p),
                                  _arr([t.shape[1] for t in dA], C.c_int32), float(rank_tol), 1 if full_q else 0,
                                  _arr([t.data_ptr() for t in dQ], C.c_void_p), _arr([t.data_ptr() for t in dR], C.c_void_p),
                                  _arr([t.data_ptr() for t in dP], C.c_void_p), rank, steps)
    N.raise_for(st, ctx)
    out = []
    for i, a in enumerate(A):
        m, c = a.shape
        kmax = min(m, c)
        FLOPS.add(2 * m * c * c)
        qcols = m if full_q else kmax
        if m == 0 or c == 0:
            Q = np.eye(m, qcols)
            R = np.zeros((kmax, c))
            perm = np.arange(c)
        else:
            Q = dQ[i].cpu().numpy()[:, :qcols]
            R = dR[i].cpu().numpy()[:kmax, :c]
            perm = dP[i].cpu().numpy()[:c].astype(np.int64)
        out.append(PivotedQR(Q=Q, R=R, perm=perm, rank=int(rank[i])))
    return out


def pivoted_qr(A, rank_tol=DEFAULT_RANK_TOL, full_q=False, device=0):
    """Householder QR with classical column-norm pivoting (reference
    densela.py:149-217): every step up to the zero-column floor, rank =
    #{|R_ii| > rank_tol |R_00|}, Q completed to m x m with full_q."""
    return pivoted_qr_batched([A], rank_tol, full_q, device)[0]


def matmul(a, b, device=0):
    """Matrix product with its 2*m*k*n flops added to the tally (reference
    densela.py:79-84), on the DMMA GEMM."""
    torch, ctx, dev = _dev(device)
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ShapeMismatchError(f"matmul: {a.shape} @ {b.shape}")
    FLOPS.add(2 * m * k * n)
    if m == 0 or n == 0:
        return np.zeros((m, n))
    da = torch.as_tensor(np.ascontiguousarray(a) if a.size else np.zeros((m, 1)), device=dev)
    db = torch.as_tensor(np.ascontiguousarray(b) if b.size else np.zeros((1, n)), device=dev)
    dc = torch.zeros((m, n), dtype=torch.float64, device=dev)
    N.order_after_torch(ctx, device)
    st = N.lib().sgf_gemm(ctx, m, n, k, 1.0, da.data_ptr(), da.shape[1], db.data_ptr(), db.shape[1], 0.0,
                          dc.data_ptr(), n)
    N.raise_for(st, ctx)
    return dc.cpu().numpy()
