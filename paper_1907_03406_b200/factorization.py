"""Drop-in `factorize` / `Preconditioner` / `RankTrace` on the B200 path.

Mirrors the reference API (`factorization.py:32-58, 73-109, 216-274,
410-573`): same argument names, defaults, validation errors, stats keys and
rank-trace format.  The host builds the partition hierarchy and the basis
(integer / tiny work, numpy) and hands them to the native library, which runs
the whole level loop on the GPU and keeps every factor in HBM.  Factor
attributes (`.idx`, `.L`, `.Q`, `.couplings`, ...) are copied back lazily on
access, for tests and inspection.
"""

from __future__ import annotations

import ctypes as C
import json
import warnings

import numpy as np

from . import _native as N
from .basis import PI_COLS_SCALAR, build_polynomial_basis
from .errors import ShapeMismatchError
from .partition import KIND_CODE, build_general_hierarchy, build_nested_hierarchy, level1_unknowns

SCHEMES = ("nest-all-all", "nest-2-all", "nest-2-2", "gen-all-all")
MODES = ("polynomial", "lowrank", "exact")
COMPRESS_KINDS = {
    "nest-all-all": ("cell1", "cell2"),
    "nest-2-all": ("cell2",),
    "nest-2-2": ("cell2",),
    "gen-all-all": ("general",),
}
UNFILTERED_KINDS = {"nest-2-2": ("cell0", "cell1")}
DEFAULT_RANK_TOL = 1e-10


def default_b(scheme, degree):
    """reference factorization.py:50-53"""
    return 3 + degree if scheme == "gen-all-all" else 3


def default_skip_levels(scheme):
    """reference factorization.py:56-58"""
    return 0 if scheme == "gen-all-all" else 2


class RankTrace(object):
    """(level, node, retained rank) triples (reference factorization.py:73-109)."""

    def __init__(self, entries=None):
        self.entries = [tuple(int(v) for v in e) for e in (entries or [])]

    def append(self, level, node, rank):
        self.entries.append((int(level), int(node), int(rank)))

    def to_json(self):
        return json.dumps({"entries": [list(e) for e in self.entries]})

    @classmethod
    def from_json(cls, text):
        return cls([tuple(e) for e in json.loads(text)["entries"]])

    def save(self, path):
        with open(path, "w") as f:
            f.write(self.to_json())

    @classmethod
    def load(cls, path):
        with open(path) as f:
            return cls.from_json(f.read())

    def __len__(self):
        return len(self.entries)

    def __eq__(self, other):
        return isinstance(other, RankTrace) and self.entries == other.entries


class _FactorView(object):
    """Lazy host view of one device factor (reference factorization.py:112-213)."""

    def __init__(self, pre, k):
        self._pre = pre
        self._k = k
        info = np.zeros(8, dtype=np.int64)
        st = N.lib().sgf_precond_factor_info(pre._h, k, info.ctypes.data)
        N.raise_for(st, pre._ctx)
        self.kind = N.FACTOR_TYPES[int(info[0])]
        self.node = None if info[0] == 2 else int(info[1])
        self.m, self.c, self.level, self.steps = int(info[2]), int(info[3]), int(info[5]), int(info[6])
        self.ncols = int(info[7])
        if info[0] == 1:
            self.retained = int(info[4])
        self._cache = {}

    def _get(self, what, shape, dtype):
        key = what
        if key not in self._cache:
            out = np.empty(shape, dtype=dtype)
            st = N.lib().sgf_precond_factor_copy(self._pre._h, self._k, what, out.ctypes.data, out.nbytes)
            N.raise_for(st, self._pre._ctx)
            self._cache[key] = out
        return self._cache[key]

    @property
    def idx(self):
        return self._get(0, (self.m,), np.int64)

    @property
    def L(self):
        return self._get(1, (self.m, self.m), np.float64)

    @property
    def Q(self):
        if self.kind != "CompressionFactor":
            raise AttributeError("Q")
        return self._get(4, (self.m, self.m), np.float64)

    @property
    def inverse_matrix(self):
        """L^{-1} (elimination / dense) or Q^T L^{-1} (compression)."""
        return self._get(5, (self.m, self.m), np.float64)

    @property
    def perm(self):
        if self.kind != "CompressionFactor":
            raise AttributeError("perm")
        return self._get(6, (self.ncols,), np.int64)

    @property
    def couplings(self):
        if self.kind != "EliminationFactor":
            raise AttributeError("couplings")
        E = self._get(2, (self.c, self.m), np.float64)
        nidx = self._get(3, (self.c,), np.int64)
        return [(nidx, E)] if self.c else []

    def _op(self, op, x):
        """One factor operation in place on a full n-vector x (a float64 numpy
        array, or a CUDA tensor on the preconditioner's device), as the
        reference's factor methods mutate their argument."""
        pre = self._pre
        if not isinstance(x, np.ndarray) and getattr(x, "is_cuda", False):
            import torch

            N.check_device_tensor(x, torch.float64, pre.device, "x")
            if x.shape != (pre.n,):
                raise ShapeMismatchError(f"expected a vector of length {pre.n}, got {tuple(x.shape)}")
            N.order_after_torch(pre._ctx, pre.device)
            N.raise_for(N.lib().sgf_factor_apply(pre._h, self._k, op, x.data_ptr(), 1), pre._ctx)
            return
        if not isinstance(x, np.ndarray) or x.dtype != np.float64 or x.shape != (pre.n,):
            raise ShapeMismatchError(f"expected a float64 numpy vector of length {pre.n}")
        buf = x if x.flags["C_CONTIGUOUS"] else np.ascontiguousarray(x)
        N.raise_for(N.lib().sgf_factor_apply(pre._h, self._k, op, buf.ctypes.data, 0), pre._ctx)
        if buf is not x:
            x[:] = buf

    def solve_forward(self, x):
        """reference factorization.py:126-130 / 173-174 / 199-200."""
        self._op(N.SOLVE_FORWARD, x)

    def solve_transpose(self, x):
        """reference factorization.py:132-136 / 176-177 / 202-203."""
        self._op(N.SOLVE_TRANSPOSE, x)

    def mult_transpose(self, x):
        """reference factorization.py:138-142 / 179-180 / 205-206."""
        self._op(N.MULT_TRANSPOSE, x)

    def mult_forward(self, x):
        """reference factorization.py:144-148 / 182-183 / 208-209."""
        self._op(N.MULT_FORWARD, x)

    def apply_flops(self):
        m = self.m
        return 4 * m * m + (4 * m * self.c if self.kind == "EliminationFactor" else 0)

    def __repr__(self):
        return f"<{self.kind} node={self.node} m={self.m} level={self.level}>"


class Preconditioner(object):
    """Ordered elementary factors resident in HBM (reference factorization.py:216-274).

    apply_inverse(x) solves A_approx y = x.  x may be a numpy array (copied to
    the device and back) or a float64 CUDA torch tensor (zero copy; a tensor is
    returned).  The object is immutable; applies are stream ordered.
    """

    def __init__(self, handle, ctx, n, stats, rank_trace, basis, scheme, degree, mode):
        # basis: a PolyBasis or a zero-argument callable building it on first use
        self._h = handle
        self._ctx = ctx
        self.n = n
        self.stats = stats
        self.rank_trace = rank_trace
        self._basis = basis
        self.scheme = scheme
        self.degree = degree
        self.mode = mode
        self._factors = None
        self.device = N.context_device(ctx)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                N.lib().sgf_precond_free(h)
            except Exception:
                pass
            self._h = None

    @property
    def basis(self):
        if callable(self._basis):
            self._basis = self._basis()
        return self._basis

    @property
    def factors(self):
        if self._factors is None:
            nf = N.lib().sgf_precond_num_factors(self._h)
            self._factors = [_FactorView(self, k) for k in range(nf)]
        return self._factors

    def _run(self, op, x):
        from .krylov import _Captured, _Probe

        if isinstance(x, _Probe):  # pcg looking inside `lambda v: P.apply_inverse(v)`
            return _Captured(self, op)
        dev = not isinstance(x, np.ndarray) and hasattr(x, "data_ptr") and getattr(x, "is_cuda", False)
        if dev:
            import torch

            if x.dtype != torch.float64 or x.dim() != 1 or x.shape[0] != self.n:
                raise ShapeMismatchError(f"expected a float64 vector of length {self.n}, got {tuple(x.shape)}")
            if x.device.index != self.device:
                raise ValueError(f"vector is on cuda:{x.device.index}, the preconditioner on cuda:{self.device}")
            xin = x.contiguous()
            y = torch.empty_like(xin)
            # the native stream must not read x before torch has written it
            N.order_after_torch(self._ctx, self.device)
            st = N.lib().sgf_apply(self._h, op, xin.data_ptr(), y.data_ptr(), 1)
            N.raise_for(st, self._ctx)
            return y
        x = np.asarray(x, dtype=float)
        if x.shape != (self.n,):
            raise ShapeMismatchError(f"expected a vector of length {self.n}, got {x.shape}")
        x = np.ascontiguousarray(x)
        y = np.empty(self.n)
        st = N.lib().sgf_apply(self._h, op, x.ctypes.data, y.ctypes.data, 0)
        N.raise_for(st, self._ctx)
        return y

    def apply_inverse(self, x):
        """W^{-T} W^{-1} x (reference :255-262)."""
        return self._run(N.APPLY_INVERSE, x)

    def apply_half_inverse(self, x):
        """W^{-1} x (reference :241-246)."""
        return self._run(N.APPLY_HALF_INVERSE, x)

    def apply_half_inverse_t(self, x):
        """W^{-T} x (reference :248-253)."""
        return self._run(N.APPLY_HALF_INVERSE_T, x)

    def apply_operator(self, x):
        """W W^T x (reference :264-271)."""
        return self._run(N.APPLY_OPERATOR, x)

    def __matmul__(self, x):
        return self.apply_inverse(x)

    def __call__(self, x):
        return self.apply_inverse(x)

    def stats_json(self):
        return json.dumps(self.stats, indent=1, sort_keys=True)


def _kind_mask(names):
    m = 0
    for k in names:
        m |= 1 << KIND_CODE[k]
    return m


def factorize(problem, scheme="nest-2-2", degree=1, b=None, skip_levels=None,
              compression=True, mode="polynomial", rank_tol=DEFAULT_RANK_TOL,
              rank_trace=None, *, replay_perms=None, device=0, device_values=None, _shard=None):
    """Build the hierarchical preconditioner on the GPU (reference
    factorization.py:410-573).  `replay_perms` (parity mode) is a list of QR
    column permutations, one per compression in the reference's execution
    order, that the device QR follows instead of its own argmax.
    `device_values` optionally supplies the CSR values (in the order of
    problem.matrix.tocsr() with sorted indices) as a float64 CUDA tensor
    already resident in HBM; the host matrix then only provides the pattern.
    `_shard` (internal, sharded.py) maps (hierarchy, skip_levels,
    compression) to the rank's sharding arguments."""
    if scheme not in SCHEMES:
        raise ValueError(f"unknown scheme {scheme!r}; expected one of {SCHEMES}")
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}; expected one of {MODES}")
    if mode == "exact":
        compression = False
    if mode == "lowrank" and compression and rank_trace is None:
        raise ValueError("mode='lowrank' requires the rank trace of a polynomial run")
    if rank_trace is not None and not (mode == "lowrank" and compression) and len(rank_trace.entries):
        # the reference iterates the trace only in low-rank mode and then
        # rejects leftover entries (factorization.py:543-549)
        raise RuntimeError(f"rank trace has {len(rank_trace.entries)} unreplayed entries; "
                           f"first: {json.dumps(list(rank_trace.entries[0]))}")
    grid = problem.grid
    n = grid.n_unknowns
    if problem.matrix.shape != (n, n):
        raise ShapeMismatchError(f"matrix is {problem.matrix.shape} but grid has {n} unknowns")
    if b is None:
        b = default_b(scheme, degree)
    if skip_levels is None:
        skip_levels = default_skip_levels(scheme)
    hier = (build_general_hierarchy if scheme == "gen-all-all" else build_nested_hierarchy)(grid, b)
    comps = grid.components_per_vertex
    if degree not in (0, 1, 2):
        raise ValueError(f"degree must be 0, 1, or 2, got {degree}")
    if comps not in (1, 3):
        raise ValueError(f"components must be 1 or 3, got {comps}")
    coords = np.ascontiguousarray(problem.coords, dtype=np.float64)
    pi_cols = PI_COLS_SCALAR[degree] * comps

    A = problem.matrix.tocsr()
    if not A.has_sorted_indices:
        A = A.copy()
        A.sort_indices()
    indptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(A.indices, dtype=np.int32)
    values = np.ascontiguousarray(A.data, dtype=np.float64)
    hl = hier.hlevels
    level_ncells = np.array([h.ncells for h in hl], dtype=np.int32)
    kinds = np.ascontiguousarray(np.concatenate([h.kind_code for h in hl]).astype(np.int8))
    interior = np.ascontiguousarray(np.concatenate([h.interior for h in hl]).astype(np.int8))
    father = (np.ascontiguousarray(np.concatenate([h.father for h in hl[:-1]]).astype(np.int64))
              if len(hl) > 1 else np.zeros(1, np.int64))
    l1_unk, l1_ptr = level1_unknowns(hier)
    l1_unk = np.ascontiguousarray(l1_unk, dtype=np.int64)
    l1_ptr = np.ascontiguousarray(l1_ptr, dtype=np.int64)

    args = N.FactorArgs()
    args.n, args.nnz = n, A.nnz
    args.indptr, args.indices, args.values = indptr.ctypes.data, indices.ctypes.data, values.ctypes.data
    args.values_on_device = 0
    if device_values is not None:
        import torch

        if tuple(device_values.shape) != (A.nnz,) or not getattr(device_values, "is_cuda", False):
            raise ShapeMismatchError("device_values must be a CUDA vector with one entry per nonzero")
        N.check_device_tensor(device_values, torch.float64, int(device), "device_values")
        args.values, args.values_on_device = device_values.data_ptr(), 1
    # Pi is built natively from the coordinates (same rule as basis.py)
    args.pi_cols, args.phi = pi_cols, None
    args.coords, args.n_vertices, args.degree, args.components = coords.ctypes.data, grid.n_vertices, degree, comps
    args.nlevels = len(hl)
    args.level_ncells = level_ncells.ctypes.data
    args.cell_kind, args.cell_interior, args.father = kinds.ctypes.data, interior.ctypes.data, father.ctypes.data
    args.l1_ptr, args.l1_unknowns = l1_ptr.ctypes.data, l1_unk.ctypes.data
    args.compress_kind_mask = _kind_mask(COMPRESS_KINDS[scheme])
    args.raw_kind_mask = _kind_mask(UNFILTERED_KINDS.get(scheme, ()))
    args.skip_levels = int(skip_levels)
    args.compression = 1 if compression else 0
    args.mode = N.MODE[mode] if compression else N.MODE["exact"]
    args.rank_tol = float(rank_tol)
    keep = []
    if mode == "lowrank" and compression:
        tr = np.ascontiguousarray(np.array(rank_trace.entries, dtype=np.int32).reshape(-1, 3))
        keep.append(tr)
        args.n_trace, args.trace = len(tr), tr.ctypes.data
    if replay_perms is not None:
        rp = np.zeros(len(replay_perms) + 1, dtype=np.int64)
        rp[1:] = np.cumsum([len(p) for p in replay_perms])
        perm_all = (np.concatenate([np.asarray(p, dtype=np.int32) for p in replay_perms])
                    if len(replay_perms) else np.zeros(1, np.int32))
        perm_all = np.ascontiguousarray(perm_all, dtype=np.int32)
        keep += [rp, perm_all]
        args.n_replay, args.replay_ptr, args.replay_perm = len(replay_perms), rp.ctypes.data, perm_all.ctypes.data
    if _shard is not None:
        sh = _shard(hier, int(skip_levels), bool(compression))
        keep.append(sh)
        args.shard_rank, args.shard_count = int(sh["rank"]), int(sh["count"])
        args.cell_rank = sh["cell_rank"].ctypes.data
        args.shard_stop_level = int(sh["stop_level"])
        args.exchange = C.cast(sh["exchange"], C.c_void_p)

    L = N.lib()
    ctx = N.context(device)
    if device_values is not None:
        N.order_after_torch(ctx, int(device))
    h = C.c_void_p()
    st = L.sgf_factorize(ctx, C.byref(args), C.byref(h))
    N.raise_for(st, ctx)
    native = json.loads(L.sgf_precond_stats_json(h).decode())
    for msg in native.get("warnings", []):
        warnings.warn(msg)
    stats = {
        "n": n, "scheme": scheme, "degree": degree,
        "mode": mode if compression else "exact",
        "b": b, "skip_levels": skip_levels,
        "levels": native["levels"], "per_level": native["per_level"],
        "max_node_size": native["max_node_size"], "max_node_seen": native["max_node_seen"],
        "final_dense_size": native["final_dense_size"],
        "flops_factorize": native["flops_factorize"], "flops_apply": native["flops_apply"],
        "peak_blocks_bytes": native["peak_blocks_bytes"], "factors": native["factors"],
    }
    nt = L.sgf_precond_rank_trace(h, None, 0)
    tr = np.zeros(max(nt, 1) * 3, dtype=np.int32)
    L.sgf_precond_rank_trace(h, tr.ctypes.data, nt)
    trace = RankTrace([tuple(int(v) for v in tr[3 * i:3 * i + 3]) for i in range(nt)])
    basis = lambda: build_polynomial_basis(problem.coords, degree, comps)  # noqa: E731
    return Preconditioner(h, ctx, n, stats, trace, basis, scheme, degree,
                          mode if compression else "exact")
