"""Device PCG with the reference recurrence (krylov.py:12-102).

`pcg(matvec, b, precond, tol, maxit, true_residual_every)` keeps the
reference signature and its operator rule (`_as_linop`, krylov.py:28-31):
`matvec` and `precond` may be matrices, `@`-able objects or callables.  The
iteration itself (dots, x/r/p updates, residual bookkeeping) always runs on
the GPU (`sgf_pcg_ops`); what varies is how an operator is applied:

* scipy sparse matrices, dense ndarrays and `DeviceCSR` -> the device CSR
  SpMV;
* a `Preconditioner`, its bound `apply_*` methods -> the device sweeps;
* a Python callable that is exactly `op @ v` / `op(v)` / `op.dot(v)` for one
  of the above (the reference's own call pattern,
  `pcg(lambda v: A @ v, b, precond=P.apply_inverse)`, bench.py:163-164) ->
  recognised by calling it once with a probe object and routed to the device
  path of `op`;
* any other callable or `@`-able object (a user operator the library cannot
  see into) -> called on host copies of the vector each iteration (a
  device->host->device round trip around the user's own code; the
  recurrence stays on the GPU).
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
        self.device = int(device)
        h = C.c_void_p()
        if A is not None:
            A = sp.csr_matrix(A)
            self._host = A  # the pattern, for callers that plan on it (sharded.pcg_sharded)
            if A.shape[0] != A.shape[1]:
                raise ShapeMismatchError(f"operator must be square, got {A.shape}")
            self.shape = A.shape
            self.n = A.shape[0]
            self.nnz = A.nnz
            ip = np.ascontiguousarray(A.indptr, dtype=np.int64)
            ix = np.ascontiguousarray(A.indices, dtype=np.int32)
            dv = np.ascontiguousarray(A.data, dtype=np.float64)
            ptrs, on_dev = (ip.ctypes.data, ix.ctypes.data, dv.ctypes.data), 0
        else:
            import torch

            self.n = int(n)
            self.shape = (self.n, self.n)
            self.nnz = int(values.shape[0])
            N.check_device_tensor(indptr, torch.int64, self.device, "indptr")
            N.check_device_tensor(indices, torch.int32, self.device, "indices")
            N.check_device_tensor(values, torch.float64, self.device, "values")
            if indptr.numel() != self.n + 1 or indices.numel() != self.nnz:
                raise ShapeMismatchError("indptr must have n+1 entries and indices one per value")
            N.order_after_torch(self._ctx)
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
        if isinstance(x, _Probe):
            return _Captured(self)
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ShapeMismatchError(f"expected a vector of length {self.n}, got {x.shape}")
        y = np.empty(self.n)
        st = N.lib().sgf_spmv(self._h, x.ctypes.data, y.ctypes.data, 0)
        N.raise_for(st, self._ctx)
        return y

    def __call__(self, x):
        return self @ x


# ---------------------------------------------------------------------------
# operator classification (reference _as_linop, krylov.py:28-31)
# ---------------------------------------------------------------------------


class _Probe(object):
    """Stand-in vector used to look inside `lambda v: op @ v`: numpy and scipy
    defer `op @ probe` to `probe.__rmatmul__`, which records `op`; the
    library's own operators record themselves.  Any other use of the probe
    fails, and the callable is then treated as opaque."""

    __array_ufunc__ = None
    __array_priority__ = 1e6

    def __rmatmul__(self, other):
        return _Captured(other)


class _Captured(object):
    def __init__(self, op, apply_op=None):
        self.op = op
        self.apply_op = apply_op


def _is_matrix(op):
    return isinstance(op, DeviceCSR) or sp.issparse(op) or (isinstance(op, np.ndarray) and op.ndim == 2)


def _capture(fn):
    """The operator behind a callable that is exactly `op @ v` (or a
    preconditioner apply), or None."""
    try:
        out = fn(_Probe())
    except Exception:
        return None
    return out if isinstance(out, _Captured) else None


class _DeviceOp(object):
    """How one operator of the solve is applied (see the module docstring).
    kind: 'csr' (device SpMV), 'precond' (device sweeps of `apply_op`),
    'host' (Python callable on host copies)."""

    def __init__(self, kind, obj, apply_op=N.APPLY_INVERSE):
        self.kind, self.obj, self.apply_op = kind, obj, apply_op


def _classify(op, role):
    from .factorization import Preconditioner

    if op is None:
        return None
    if isinstance(op, Preconditioner):
        return _DeviceOp("precond", op)
    owner = getattr(op, "__self__", None)
    name = getattr(op, "__name__", "")
    if isinstance(owner, Preconditioner) and name in _APPLY_NAMES:
        return _DeviceOp("precond", owner, _APPLY_NAMES[name])
    if _is_matrix(op):
        return _DeviceOp("csr", op)
    fn = op if callable(op) else (lambda x: op @ x)
    cap = _capture(fn)
    if cap is not None:
        if isinstance(cap.op, Preconditioner):
            return _DeviceOp("precond", cap.op, cap.apply_op if cap.apply_op is not None else N.APPLY_INVERSE)
        if _is_matrix(cap.op):
            return _DeviceOp("csr", cap.op)
    return _DeviceOp("host", fn)


_APPLY_NAMES = {"apply_inverse": N.APPLY_INVERSE, "__call__": N.APPLY_INVERSE, "__matmul__": N.APPLY_INVERSE,
                "apply_half_inverse": N.APPLY_HALF_INVERSE, "apply_half_inverse_t": N.APPLY_HALF_INVERSE_T,
                "apply_operator": N.APPLY_OPERATOR}


def _solve_device(A, M):
    """The device of the solve: the preconditioner's, else the matrix's."""
    for op in (M, A):
        if op is None:
            continue
        if op.kind == "precond":
            return N.context_device(op.obj._ctx)
        if op.kind == "csr" and isinstance(op.obj, DeviceCSR):
            return op.obj.device
    return 0


class _Callbacks(object):
    """ctypes callbacks for the operators that are not the solve's own CSR or
    preconditioner handle; keeps them (and the first Python exception raised
    inside one) alive for the duration of the call."""

    def __init__(self, ctx, n):
        self.ctx, self.n = ctx, n
        self.errors = []
        self.keep = []

    def _guard(self, body):
        def cb(user, pin, pout):
            try:
                body(pin, pout)
                return 0
            except BaseException as e:  # noqa: BLE001 - re-raised after the native call returns
                self.errors.append(e)
                return N.SGF_INVALID_ARG
        f = N.PRECOND_FN(cb)
        self.keep.append(f)
        return f

    def device_csr(self, csr):
        L = N.lib()
        return self._guard(lambda pin, pout: N.raise_for(L.sgf_spmv(csr._h, pin, pout, 1), csr._ctx))

    def device_precond(self, P, op):
        L = N.lib()
        return self._guard(lambda pin, pout: N.raise_for(L.sgf_apply(P._h, op, pin, pout, 1), P._ctx))

    def host(self, fn):
        n, ctx, L = self.n, self.ctx, N.lib()
        buf = np.empty(n)

        def body(pin, pout):
            N.raise_for(L.sgf_memcpy(ctx, buf.ctypes.data, pin, 8 * n), ctx)
            y = np.ascontiguousarray(np.asarray(fn(buf.copy()), dtype=np.float64))
            if y.shape != (n,):
                raise ShapeMismatchError(f"operator returned shape {y.shape}, expected ({n},)")
            N.raise_for(L.sgf_memcpy(ctx, pout, y.ctypes.data, 8 * n), ctx)
        return self._guard(body)


def pcg(matvec, b, precond=None, tol=1e-10, maxit=5000, true_residual_every=50):
    """Conjugate gradients (reference krylov.py:34-102) with the recurrence
    on the GPU.  With a float64 CUDA tensor `b` the solve stays on the
    device and x is returned as a CUDA tensor."""
    on_dev = not isinstance(b, np.ndarray) and getattr(b, "is_cuda", False)
    if not on_dev:
        b = np.asarray(b, dtype=float)
        if b.ndim != 1:
            raise ShapeMismatchError(f"right-hand side must be a vector, got {b.shape}")
    elif b.dim() != 1:
        raise ShapeMismatchError(f"right-hand side must be a vector, got {tuple(b.shape)}")
    n = int(b.shape[0])
    Aop = _classify(matvec, "matvec")
    if Aop is None:
        raise TypeError("pcg needs an operator")
    Mop = _classify(precond, "precond")
    dev = _solve_device(Aop, Mop)
    ctx = N.context(dev)
    cbs = _Callbacks(ctx, n)
    L = N.lib()
    # the operator: the solve's own CSR when it is a matrix, else a callback
    a_h, mv = None, N.MATVEC_FN()
    if Aop.kind == "csr":
        csr = Aop.obj if isinstance(Aop.obj, DeviceCSR) and Aop.obj.device == dev else DeviceCSR(
            Aop.obj if not isinstance(Aop.obj, DeviceCSR) else _host_csr(Aop.obj), device=dev)
        if csr.n != n:
            raise ShapeMismatchError(f"matrix is {csr.shape}, rhs has {n} entries")
        a_h = csr._h
        cbs.keep.append(csr)
    elif Aop.kind == "precond":
        if Aop.obj.n != n:
            raise ShapeMismatchError(f"operator has {Aop.obj.n} rows, rhs has {n} entries")
        mv = cbs.device_precond(Aop.obj, Aop.apply_op)
    else:
        mv = cbs.host(Aop.obj)
    p_h, pf = None, N.PRECOND_FN()
    if Mop is not None:
        if Mop.kind == "precond":
            if Mop.obj.n != n:
                raise ShapeMismatchError(f"preconditioner has {Mop.obj.n} rows, rhs has {n} entries")
            if N.context_device(Mop.obj._ctx) != dev:
                raise ValueError("the preconditioner lives on another device than the solve")
            if Mop.apply_op == N.APPLY_INVERSE:
                p_h = Mop.obj._h
            else:
                pf = cbs.device_precond(Mop.obj, Mop.apply_op)
        elif Mop.kind == "csr":
            mcsr = Mop.obj if isinstance(Mop.obj, DeviceCSR) and Mop.obj.device == dev else DeviceCSR(
                Mop.obj if not isinstance(Mop.obj, DeviceCSR) else _host_csr(Mop.obj), device=dev)
            if mcsr.n != n:
                raise ShapeMismatchError(f"preconditioner is {mcsr.shape}, rhs has {n} entries")
            cbs.keep.append(mcsr)
            pf = cbs.device_csr(mcsr)
        else:
            pf = cbs.host(Mop.obj)
    hist = np.empty(int(maxit) + 2)
    rep = N.PcgReport()
    if on_dev:
        import torch

        if b.dtype != torch.float64 or b.device.index != dev:
            raise ShapeMismatchError(f"right-hand side must be a float64 vector on cuda:{dev}")
        b = b.contiguous()
        x = torch.empty_like(b)
        N.order_after_torch(ctx, dev)
        bp, xp = b.data_ptr(), x.data_ptr()
    else:
        b = np.ascontiguousarray(b)
        x = np.empty_like(b)
        bp, xp = b.ctypes.data, x.ctypes.data
    st = L.sgf_pcg_ops(ctx, n, a_h, mv, None, p_h, pf, None, bp, xp, float(tol), int(maxit),
                       int(true_residual_every), 1 if on_dev else 0, C.byref(rep), hist.ctypes.data)
    if cbs.errors:
        raise cbs.errors[0]
    N.raise_for(st, ctx)
    return x, SolveReport(iterations=rep.iterations, residual_history=hist[:rep.history_len].tolist(),
                          converged=bool(rep.converged), wall_time=rep.wall_time,
                          final_rel_residual=rep.final_rel_residual)


def _host_csr(A):
    raise ValueError(f"DeviceCSR on cuda:{A.device} cannot serve a solve on another device")
