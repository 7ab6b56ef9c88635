"""Multi-GPU factorize -> apply -> PCG: one process per GPU, subtree sharding
of the nested-dissection tree (north star item 4).

Partition.  Pick the partition level p = (first level that compresses) + 1
(or the top level when nothing compresses).  Its interior cells ("octants":
the 8 regions cut out by the top separator planes at 128^3) and all their
descendants are assigned to ranks in contiguous blocks; level-1 cells whose
level-p ancestor is a separator are top-separator cells, shared by all.
Interiors at levels < p never lie on a level-p separator, so every
elimination of the local phase (levels 1 .. p-1) belongs to exactly one rank
and touches only that rank's cells and top-separator cells.

Factorization.  Every rank runs the same symbolic level loop (identical block
table, fill, flop and byte tallies -- the structure is value-independent until
the first compression) and computes the eliminations of its own
interiors; a block gets the matrix entries on exactly one rank (its owned
cell's rank, rank 0 for top-separator pairs).  At the end of the local phase
the trailing-matrix block regions, laid out identically on every rank, are
summed onto rank 0 with one reduction per region (NCCL over NVLink), and rank
0 continues with the compressions, the top levels and the dense factor.
Shared blocks thus receive  A + sum_r (sum of rank r's Schur updates)
instead of the reference's ascending-interior sequence: a rounding-level
change, deterministic run to run.

Apply (collective).  Vectors are replicated.  Each rank runs the forward
sweeps of its local factors; the changes of the top unknowns are summed onto
rank 0, which runs the top forward and backward sweeps and broadcasts the top
unknowns; each rank runs its local backward sweeps; the disjoint pieces are
assembled with one all-reduce (exactly one nonzero contribution per entry).

PCG.  The native PCG (same recurrence as krylov.pcg) runs on every rank with
replicated vectors and the sharded apply as a callback; SpMV and dot products
are computed redundantly per rank (a 128^3 SpMV is ~50 us on one GPU, below
the cost of a halo exchange round at this size), so every rank takes the same
branches without extra communication.

Communication goes through torch.distributed: NCCL on GPUs; with the gloo
backend (CPU tests, or several ranks sharing one GPU in the parity test) the
device buffers are staged through host memory.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .errors import ShapeMismatchError
from .krylov import DeviceCSR, SolveReport


# ---------------------------------------------------------------------------
# partition (pure host logic; tested with gloo on CPU)
# ---------------------------------------------------------------------------
def shard_plan(hier, nranks, skip_levels, compression):
    """Level-1 cell ownership for `nranks` ranks.

    Returns (cell_rank int32[ncells_L1], stop_level, partition_level) with
    cell_rank = -1 for top-separator cells.  stop_level is the last level of
    the local phase (1-based)."""
    hl = hier.hlevels
    nlev = len(hl)
    first_comp = skip_levels + 1 if compression else nlev
    # partition level, 1-based: the level after the last compression-free
    # level, lowered until it has at least two interior cells (regions)
    p = min(max(first_comp, 1) + 1, nlev)
    while p > 2 and int(np.count_nonzero(hl[p - 1].interior)) < 2:
        p -= 1
    stop = p - 1
    nc1 = hl[0].ncells
    if stop < 1 or nranks <= 1:
        return np.zeros(nc1, np.int32), 1, 1  # everything on rank 0
    # level-1 cell -> its level-p ancestor
    anc = np.arange(nc1, dtype=np.int64)
    for t in range(p - 1):
        anc = np.asarray(hl[t].father, dtype=np.int64)[anc]
    top = hl[p - 1]
    octants = np.flatnonzero(top.interior)
    if octants.size == 0:
        return np.zeros(nc1, np.int32), stop, p
    orank = np.full(top.ncells, -1, dtype=np.int32)
    orank[octants] = (np.arange(octants.size) * nranks) // octants.size
    cell_rank = orank[anc].astype(np.int32)
    check_plan(hier, cell_rank, stop)
    return np.ascontiguousarray(cell_rank), stop, p


def check_plan(hier, cell_rank, stop):
    """Every interior eliminated in the local phase (levels 1..stop) must be
    owned by exactly one rank: all its level-1 descendants share one rank >= 0."""
    hl = hier.hlevels
    r = np.asarray(cell_rank, dtype=np.int64)
    for t in range(stop):
        h = hl[t]
        bad = h.interior & (r < 0)
        if bad.any():
            raise ValueError(f"level {t + 1}: interior cell {int(np.flatnonzero(bad)[0])} has no owning rank")
        if t + 1 < len(hl):
            f = np.asarray(h.father, dtype=np.int64)
            nf = hl[t + 1].ncells
            lo = np.full(nf, np.iinfo(np.int64).max)
            hi = np.full(nf, np.iinfo(np.int64).min)
            np.minimum.at(lo, f, r)
            np.maximum.at(hi, f, r)
            used = lo <= hi
            if np.any(lo[used] != hi[used]):
                raise ValueError(f"level {t + 2}: a cell has children on different ranks")
            nr = np.full(nf, -1, dtype=np.int64)
            nr[used] = lo[used]
            r = nr


# ---------------------------------------------------------------------------
# communication helpers (torch.distributed; gloo stages through the host)
# ---------------------------------------------------------------------------
def _dist():
    import torch.distributed as dist

    return dist


def _is_gloo(group=None):
    return _dist().get_backend(group) == "gloo"


def _reduce_sum(t, group=None):
    dist = _dist()
    if _is_gloo(group) and t.is_cuda:
        h = t.cpu()
        dist.reduce(h, dst=0, op=dist.ReduceOp.SUM, group=group)
        if dist.get_rank(group) == 0:
            t.copy_(h)
    else:
        dist.reduce(t, dst=0, op=dist.ReduceOp.SUM, group=group)


def _broadcast(t, group=None):
    dist = _dist()
    if _is_gloo(group) and t.is_cuda:
        h = t.cpu()
        dist.broadcast(h, src=0, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src=0, group=group)


def _allreduce_sum(t, group=None):
    dist = _dist()
    if _is_gloo(group) and t.is_cuda:
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


class _DevBuf:
    """__cuda_array_interface__ view of a raw float64 device buffer."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _wrap(ptr, count, device):
    import torch

    return torch.as_tensor(_DevBuf(ptr, count), device=device)


def _stream(ctx, device):
    import torch

    return torch.cuda.ExternalStream(N.lib().sgf_stream(ctx), device=device)


# ---------------------------------------------------------------------------
# sharded preconditioner
# ---------------------------------------------------------------------------
class ShardedPreconditioner:
    """One rank's share of a preconditioner factorized across a process group.
    apply_inverse is collective (every rank calls it with the same vector)."""

    def __init__(self, pre, group, device):
        import torch

        self.pre = pre
        self.n = pre.n
        self.group = group
        self.device = device
        dist = _dist()
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        L = N.lib()
        nlf, nlu, ntop = C.c_int64(), C.c_int64(), C.c_int64()
        N.raise_for(L.sgf_precond_shard_info(pre._h, C.byref(nlf), C.byref(nlu), C.byref(ntop)), pre._ctx)
        loc = np.zeros(max(nlu.value, 1), np.int64)
        N.raise_for(L.sgf_precond_shard_set(pre._h, 0, loc.ctypes.data, loc.size), pre._ctx)
        top = np.zeros(max(ntop.value, 1), np.int64)
        N.raise_for(L.sgf_precond_shard_set(pre._h, 1, top.ctypes.data, top.size), pre._ctx)
        self.n_local_factors = nlf.value
        self.local_idx = torch.as_tensor(loc[:nlu.value], device=device)
        self.top_idx = torch.as_tensor(top[:ntop.value], device=device)
        self.stream = _stream(pre._ctx, device)
        self.stats = pre.stats if self.rank == 0 else None
        self.rank_trace = pre.rank_trace if self.rank == 0 else None

    def _part(self, part, y):
        N.raise_for(N.lib().sgf_apply_part(self.pre._h, part, y.data_ptr()), self.pre._ctx)

    def apply_into(self, x, out):
        """out = M^-1 x on device tensors (enqueued on the native stream)."""
        import torch

        with torch.cuda.stream(self.stream):
            y = x.clone()
            self._part(0, y)                        # local forward sweeps
            top = self.top_idx
            d = y[top] - x[top]                     # this rank's updates of the top unknowns
            _reduce_sum(d, self.group)
            if self.rank == 0:
                y[top] = x[top] + d
                self._part(1, y)                    # top forward + backward sweeps
                t = y[top]
            else:
                t = torch.empty_like(d)
            _broadcast(t, self.group)
            y[top] = t
            self._part(2, y)                        # local backward sweeps
            out.zero_()
            out[self.local_idx] = y[self.local_idx]
            if self.rank == 0:
                out[top] = t
            _allreduce_sum(out, self.group)
        return out

    def apply_inverse(self, x):
        import torch

        dev = not isinstance(x, np.ndarray) and getattr(x, "is_cuda", False)
        xt = x if dev else torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=self.device)
        if xt.dtype != torch.float64 or xt.shape != (self.n,):
            raise ShapeMismatchError(f"expected a float64 vector of length {self.n}, got {tuple(xt.shape)}")
        out = torch.empty_like(xt)
        self.apply_into(xt, out)
        self.stream.synchronize()
        return out if dev else out.cpu().numpy()

    __call__ = apply_inverse


def factorize_sharded(problem, group=None, device=None, **kw):
    """Collective factorize across the ranks of `group` (default: the world).
    Accepts the keyword arguments of factorize(); returns this rank's
    ShardedPreconditioner (rank 0 holds the stats and the rank trace)."""
    import torch

    from .factorization import factorize

    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if device is None:
        device = torch.cuda.current_device()
    dev = torch.device("cuda", device)
    ctx = N.context(device)
    stream = _stream(ctx, dev)

    def exchange(user, nregions, ptrs, counts):
        try:
            with torch.cuda.stream(stream):
                for i in range(nregions):
                    _reduce_sum(_wrap(ptrs[i], counts[i], dev), group)
            stream.synchronize()
            return 0
        except Exception as e:  # surfaces as a factorize failure
            import sys

            print(f"[sharded] exchange failed on rank {rank}: {e!r}", file=sys.stderr)
            return 1

    cb = N.EXCHANGE_FN(exchange)

    def shard(hier, skip_levels, compression):
        cell_rank, stop, _ = shard_plan(hier, world, skip_levels, compression)
        return {"rank": rank, "count": max(world, 2), "cell_rank": cell_rank, "stop_level": stop,
                "exchange": cb}

    pre = factorize(problem, device=device, _shard=shard, **kw)
    return ShardedPreconditioner(pre, group, dev)


def pcg_sharded(A, b, precond, tol=1e-10, maxit=5000, true_residual_every=50):
    """Collective PCG (reference krylov.py:34-102) with a ShardedPreconditioner;
    A is a DeviceCSR (or a scipy matrix) on every rank, b the same vector on
    every rank (numpy or a CUDA tensor).  Returns (x, SolveReport) on every rank."""
    import torch

    if not isinstance(A, DeviceCSR):
        A = DeviceCSR(A, device=precond.device.index)
    n = A.n
    if precond.n != n:
        raise ShapeMismatchError("preconditioner and matrix sizes differ")
    dev = not isinstance(b, np.ndarray) and getattr(b, "is_cuda", False)
    bt = b if dev else torch.as_tensor(np.ascontiguousarray(b, dtype=np.float64), device=precond.device)
    x = torch.empty_like(bt)
    err = []

    def cb(user, pin, pout):
        try:
            precond.apply_into(_wrap(pin, n, precond.device), _wrap(pout, n, precond.device))
            return 0
        except Exception as e:
            err.append(e)
            return N.SGF_CUDA

    fn = N.PRECOND_FN(cb)
    rep = N.PcgReport()
    hist = np.zeros(maxit + 2)
    st = N.lib().sgf_pcg_cb(A._ctx, A._h, fn, None, bt.data_ptr(), x.data_ptr(), float(tol), int(maxit),
                            int(true_residual_every), 1, C.byref(rep), hist.ctypes.data)
    if err:
        raise err[0]
    N.raise_for(st, A._ctx)
    report = SolveReport(iterations=rep.iterations, residual_history=hist[:rep.history_len].tolist(),
                         converged=bool(rep.converged), wall_time=rep.wall_time,
                         final_rel_residual=rep.final_rel_residual)
    return (x if dev else x.cpu().numpy()), report
