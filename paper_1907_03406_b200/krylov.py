"""Device PCG with the reference recurrence (krylov.py:12-102).

`pcg(matvec, b, precond, tol, maxit, true_residual_every)` keeps the
reference signature.  The whole iteration runs on the GPU: CSR SpMV,
fixed-order dot products, fused x/r updates and the level-batched
preconditioner sweeps.  `matvec` must be a sparse matrix (scipy CSR/CSC/COO,
or a `DeviceCSR`), `precond` a `Preconditioner` (or its bound
`apply_inverse`) or None; arbitrary Python callables are rejected instead of
being silently run on the CPU.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _native as N
from .errors import ShapeMismatchError


@dataclass
class SolveReport:
    iterations: int
    residual_history: list = field(default_factory=list)
    converged: bool = False
    wall_time: float = 0.0
    final_rel_residual: float = 0.0


class DeviceCSR(object):
    """A CSR matrix resident in HBM (int32 column indices, int64 row pointer)."""

    def __init__(self, A=None, device=0, *, indptr=None, indices=None, values=None, n=None):
        """From a scipy matrix (host), or from CUDA tensors indptr (int64),
        indices (int32) and values (float64) already resident in HBM."""
        self._ctx = N.context(device)
        h = C.c_void_p()
        if A is not None:
            A = sp.csr_matrix(A)
            self.shape = A.shape
            self.n = A.shape[0]
            self.nnz = A.nnz
            ip = np.ascontiguousarray(A.indptr, dtype=np.int64)
            ix = np.ascontiguousarray(A.indices, dtype=np.int32)
            dv = np.ascontiguousarray(A.data, dtype=np.float64)
            ptrs, on_dev = (ip.ctypes.data, ix.ctypes.data, dv.ctypes.data), 0
        else:
            self.n = int(n)
            self.shape = (self.n, self.n)
            self.nnz = int(values.shape[0])
            ptrs, on_dev = (indptr.data_ptr(), indices.data_ptr(), values.data_ptr()), 1
        st = N.lib().sgf_csr_create(self._ctx, self.n, self.nnz, ptrs[0], ptrs[1], ptrs[2], on_dev, C.byref(h))
        N.raise_for(st, self._ctx)
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                N.lib().sgf_csr_free(h)
            except Exception:
                pass
            self._h = None

    def __matmul__(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ShapeMismatchError(f"expected a vector of length {self.n}, got {x.shape}")
        y = np.empty(self.n)
        st = N.lib().sgf_spmv(self._h, x.ctypes.data, y.ctypes.data, 0)
        N.raise_for(st, self._ctx)
        return y


def _as_device_matrix(matvec):
    if isinstance(matvec, DeviceCSR):
        return matvec
    if sp.issparse(matvec):
        # a host matrix is uploaded per call (keep a DeviceCSR to reuse it)
        return DeviceCSR(matvec)
    raise TypeError("pcg needs the operator as a sparse matrix (scipy.sparse or DeviceCSR) so the "
                    "iteration can run on the GPU; Python callables are not executed on the host")


def _as_device_precond(precond):
    from .factorization import Preconditioner

    if precond is None:
        return None
    if isinstance(precond, Preconditioner):
        return precond
    owner = getattr(precond, "__self__", None)
    if isinstance(owner, Preconditioner) and getattr(precond, "__name__", "") == "apply_inverse":
        return owner
    raise TypeError("precond must be a Preconditioner (or its apply_inverse) produced by factorize()")


def pcg(matvec, b, precond=None, tol=1e-10, maxit=5000, true_residual_every=50):
    """Conjugate gradients (reference krylov.py:34-102) on the GPU.  With a
    float64 CUDA tensor `b` the solve stays on the device and x is returned
    as a CUDA tensor."""
    if not isinstance(b, np.ndarray) and getattr(b, "is_cuda", False):
        import torch

        A = _as_device_matrix(matvec)
        P = _as_device_precond(precond)
        if b.dim() != 1 or b.shape[0] != A.n or b.dtype != torch.float64:
            raise ShapeMismatchError(f"right-hand side must be a float64 vector of length {A.n}")
        b = b.contiguous()
        x = torch.empty_like(b)
        hist = np.empty(int(maxit) + 2)
        rep = N.PcgReport()
        st = N.lib().sgf_pcg(A._ctx, A._h, P._h if P is not None else None, b.data_ptr(), x.data_ptr(),
                             float(tol), int(maxit), int(true_residual_every), 1, C.byref(rep),
                             hist.ctypes.data)
        N.raise_for(st, A._ctx)
        return x, SolveReport(iterations=rep.iterations, residual_history=hist[:rep.history_len].tolist(),
                              converged=bool(rep.converged), wall_time=rep.wall_time,
                              final_rel_residual=rep.final_rel_residual)
    b = np.asarray(b, dtype=float)
    if b.ndim != 1:
        raise ShapeMismatchError(f"right-hand side must be a vector, got {b.shape}")
    A = _as_device_matrix(matvec)
    P = _as_device_precond(precond)
    if A.n != b.shape[0]:
        raise ShapeMismatchError(f"matrix is {A.shape}, rhs has {b.shape[0]} entries")
    b = np.ascontiguousarray(b)
    x = np.empty_like(b)
    hist = np.empty(int(maxit) + 2)
    rep = N.PcgReport()
    st = N.lib().sgf_pcg(A._ctx, A._h, P._h if P is not None else None, b.ctypes.data, x.ctypes.data,
                         float(tol), int(maxit), int(true_residual_every), 0, C.byref(rep), hist.ctypes.data)
    N.raise_for(st, A._ctx)
    return x, SolveReport(iterations=rep.iterations, residual_history=hist[:rep.history_len].tolist(),
                          converged=bool(rep.converged), wall_time=rep.wall_time,
                          final_rel_residual=rep.final_rel_residual)
