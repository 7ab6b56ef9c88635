"""Multi-GPU factorize -> apply -> PCG: one process per GPU, subtree sharding
of the nested-dissection tree (north star item 4).

Partition (`shard_plan`).  The local phase covers the eliminations of levels
1 .. stop, stop = the first compressing level (its eliminations run before
its compressions, factorization.py:483-490; compressions need the summed
separator blocks, so they come after the exchange).  The partition cells are
the interior cells of level stop + 1 when it has at least two ("octants": the
8 regions cut out by the top separator planes at 128^3, b = 9), else the
interiors of level `stop` itself (BASELINE cfg2: its 8 level-3 nodes of
2654-3571 unknowns, 71.5% of the flops, are eliminated on their owners).  A
partition cell and all its descendants belong to one rank (contiguous blocks
of cells per rank); level-1 cells whose partition-level ancestor is a
separator are top-separator cells, shared.  Every local elimination has
exactly one owner and touches only its owner's cells and top-separator cells
(`check_plan`).

Factorization.  Every rank runs the same symbolic level loop (identical block
table, fill, flop and byte tallies: the structure is value-independent until
the first compression) and computes its own interiors; a block
gets the matrix entries on one rank (its owned cell's rank, rank 0 for
top-separator pairs).  At the end of the local phase each rank packs the
trailing-matrix blocks it holds nonzero data for -- its own cells' blocks and
its partial Schur sums of shared blocks -- and rank 0 receives every other
rank's package and adds it in ascending rank order (native
`sgf_exchange_accumulate`); nothing else moves.  Rank 0 continues with the
compressions, the top levels and the dense factor.  Shared blocks thus hold
A + sum_r (rank r's Schur updates) instead of the reference's
ascending-interior sequence: a rounding-level change, deterministic run to
run.  `ShardedPreconditioner.exchange_log` records what was sent.

Apply (collective, `sgf_apply_shard`).  Vectors are distributed: a rank owns
the unknowns its local factors eliminate, rank 0 also the top unknowns.
Stage 0: local forward sweeps, the changes of the top unknowns packed natively
-> summed onto rank 0; stage 1 (rank 0): top forward + backward sweeps -> the
top unknowns broadcast; stage 2: local backward sweeps, non-owned entries
zeroed.  The collectives move only the top-unknown buffer.

PCG (`pcg_sharded`, native `sgf_pcg_dist`).  The reference recurrence on
distributed vectors: SpMV over the rank's owned rows after a halo exchange
(the owned entries of other ranks that those rows reference; with the octant
partition every rank talks only to rank 0), inner products as local partials
all-gathered and summed in rank order (bitwise identical on every rank, so
every rank takes the same branches), the sharded apply as preconditioner.

Communication goes through torch.distributed: NCCL on GPUs; with the gloo
backend (CPU tests, or several ranks sharing one GPU in the parity tests)
device buffers are staged through host memory.  torch is plumbing here:
buffers and collectives; every arithmetic step is a native kernel.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.sparse as sp

from . import _native as N
from .errors import ShapeMismatchError
from .krylov import DeviceCSR, SolveReport


# ---------------------------------------------------------------------------
# partition (pure host logic; tested with gloo on CPU)
# ---------------------------------------------------------------------------
def shard_plan(hier, nranks, skip_levels, compression):
    """Level-1 cell ownership for `nranks` ranks.

    Returns (cell_rank int32[ncells_L1], stop_level, partition_level) with
    cell_rank = -1 for top-separator cells; stop_level is the last level
    whose eliminations run in the local phase (1-based)."""
    hl = hier.hlevels
    nlev = len(hl)
    nc1 = hl[0].ncells

    def interiors(level):
        return int(np.count_nonzero(hl[level - 1].interior)) if 1 <= level <= nlev else 0

    first_comp = skip_levels + 1 if compression else nlev
    stop = min(max(first_comp, 1), nlev - 1)   # the single top cell is the dense factor
    p = 0
    while stop >= 1:
        if interiors(stop + 1) >= 2 and stop + 1 < nlev:
            p = stop + 1
            break
        if interiors(stop) >= 2:
            p = stop
            break
        stop -= 1
    if stop < 1 or p < 1 or nranks <= 1:
        return np.zeros(nc1, np.int32), max(stop, 1), max(p, 1)
    # level-1 cell -> its partition-level ancestor
    anc = np.arange(nc1, dtype=np.int64)
    for t in range(p - 1):
        anc = np.asarray(hl[t].father, dtype=np.int64)[anc]
    part = hl[p - 1]
    cells = np.flatnonzero(part.interior)
    orank = np.full(part.ncells, -1, dtype=np.int32)
    orank[cells] = (np.arange(cells.size) * nranks) // cells.size
    cell_rank = orank[anc].astype(np.int32)
    check_plan(hier, cell_rank, stop)
    return np.ascontiguousarray(cell_rank), stop, p


def check_plan(hier, cell_rank, stop):
    """Every interior eliminated in the local phase (levels 1..stop) is owned
    by exactly one rank: all its level-1 descendants share one rank >= 0."""
    hl = hier.hlevels
    r = np.asarray(cell_rank, dtype=np.int64)
    for t in range(stop):
        h = hl[t]
        bad = h.interior & (r < 0)
        if bad.any():
            raise ValueError(f"level {t + 1}: interior cell {int(np.flatnonzero(bad)[0])} has no owning rank")
        if t + 1 >= min(stop, len(hl)):
            break  # the ranks of cells above the last local level are not used
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


def _comm(t, group=None):
    """The tensor to hand to a collective: host copy under gloo."""
    return t.cpu() if (_is_gloo(group) and t.is_cuda) else t


def _reduce_sum(t, group=None):
    dist = _dist()
    h = _comm(t, group)
    dist.reduce(h, dst=0, op=dist.ReduceOp.SUM, group=group)
    if h is not t and dist.get_rank(group) == 0:
        t.copy_(h)


def _broadcast(t, group=None):
    dist = _dist()
    h = _comm(t, group)
    dist.broadcast(h, src=0, group=group)
    if h is not t:
        t.copy_(h)


def _allreduce_sum(t, group=None):
    dist = _dist()
    h = _comm(t, group)
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    if h is not t:
        t.copy_(h)


def _send(t, dst, group=None):
    dist = _dist()
    dist.send(_comm(t, group), dst=dist.get_global_rank(group, dst) if group is not None else dst, group=group)


def _recv(t, src, group=None):
    dist = _dist()
    h = _comm(t, group)
    dist.recv(h, src=dist.get_global_rank(group, src) if group is not None else src, group=group)
    if h is not t:
        t.copy_(h)


def _sum_in_rank_order(vals, group=None, device=None):
    """Sum a few doubles across ranks, adding the ranks' values in ascending
    rank order: bitwise the same result on every rank."""
    import torch

    dist = _dist()
    world = dist.get_world_size(group)
    v = torch.as_tensor(np.asarray(vals, dtype=np.float64))
    if not _is_gloo(group):
        v = v.to(device)
    outs = [torch.empty_like(v) for _ in range(world)]
    dist.all_gather(outs, v, group=group)
    acc = outs[0].cpu().numpy().copy()
    for o in outs[1:]:
        acc += o.cpu().numpy()
    return acc


class _DevBuf:
    """__cuda_array_interface__ view of a raw device buffer."""

    def __init__(self, ptr, count, typestr="<f8"):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _wrap(ptr, count, device, typestr="<f8"):
    import torch

    return torch.as_tensor(_DevBuf(ptr, count, typestr), device=device)


def _stream(ctx, device):
    import torch

    return torch.cuda.ExternalStream(N.lib().sgf_stream(ctx), device=device)


# ---------------------------------------------------------------------------
# sharded preconditioner
# ---------------------------------------------------------------------------
class ShardedPreconditioner:
    """One rank's share of a preconditioner factorized across a process group.
    apply_inverse is collective (every rank calls it with the same vector)."""

    def __init__(self, pre, group, device, exchange_log, plan):
        import torch

        self.pre = pre
        self.n = pre.n
        self.group = group
        self.device = device
        dist = _dist()
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.exchange_log = exchange_log
        self.plan = plan
        L = N.lib()
        nlf, nlu, ntop = C.c_int64(), C.c_int64(), C.c_int64()
        N.raise_for(L.sgf_precond_shard_info(pre._h, C.byref(nlf), C.byref(nlu), C.byref(ntop)), pre._ctx)
        loc = np.zeros(max(nlu.value, 1), np.int64)
        N.raise_for(L.sgf_precond_shard_set(pre._h, 0, loc.ctypes.data, loc.size), pre._ctx)
        top = np.zeros(max(ntop.value, 1), np.int64)
        N.raise_for(L.sgf_precond_shard_set(pre._h, 1, top.ctypes.data, top.size), pre._ctx)
        self.n_local_factors = nlf.value
        self.local_idx = loc[:nlu.value].copy()
        self.top_idx = top[:ntop.value].copy()
        self.owned = np.sort(np.concatenate([self.local_idx, self.top_idx]) if self.rank == 0 else self.local_idx)
        self.top_buf = torch.empty(max(ntop.value, 1), dtype=torch.float64, device=device)
        self.stream = _stream(pre._ctx, device)
        self.stats = pre.stats if self.rank == 0 else None
        self.rank_trace = pre.rank_trace if self.rank == 0 else None

    def masked(self, x):
        """This rank's owned entries of a replicated device vector, zeros
        elsewhere (native gather + scatter)."""
        import torch

        if getattr(self, "_own", None) is None:
            self._own = torch.as_tensor(self.owned.astype(np.int32), device=self.device)
            self._tmp = torch.empty(max(len(self.owned), 1), dtype=torch.float64, device=self.device)
        xm = torch.zeros_like(x)
        L, ctx, k = N.lib(), self.pre._ctx, len(self.owned)
        N.order_after_torch(ctx, self.device.index)
        N.raise_for(L.sgf_vec_gather(ctx, x.data_ptr(), self._own.data_ptr(), self._tmp.data_ptr(), k), ctx)
        N.raise_for(L.sgf_vec_scatter(ctx, self._tmp.data_ptr(), self._own.data_ptr(), xm.data_ptr(), k), ctx)
        return xm

    def _stage(self, stage, x_ptr, y_ptr, mask=1):
        N.order_after_torch(self.pre._ctx, self.device.index)  # after the collective on top_buf
        N.raise_for(N.lib().sgf_apply_shard(self.pre._h, stage, x_ptr, y_ptr, self.top_buf.data_ptr(), mask),
                    self.pre._ctx)

    def apply_dist(self, x_ptr, y_ptr):
        """y = M^-1 x on distributed device vectors (raw pointers, n doubles:
        owned entries meaningful, the rest zero)."""
        t = self.top_buf[:len(self.top_idx)]
        self._stage(0, x_ptr, y_ptr)                 # local forward sweeps, top changes packed
        if len(self.top_idx):
            _reduce_sum(t, self.group)
        if self.rank == 0:
            self._stage(1, x_ptr, y_ptr)             # top forward + backward sweeps
        if len(self.top_idx):
            _broadcast(t, self.group)
        self._stage(2, x_ptr, y_ptr)                 # local backward sweeps, non-owned entries zeroed

    def apply_into(self, x, out):
        """out = M^-1 x for a vector replicated on every rank (device tensors):
        distributed apply, then one all-reduce assembles the owned pieces."""
        import torch

        xm = self.masked(x)
        self.apply_dist(xm.data_ptr(), out.data_ptr())
        _allreduce_sum(out, self.group)
        return out

    def apply_inverse(self, x):
        import torch

        dev = not isinstance(x, np.ndarray) and getattr(x, "is_cuda", False)
        xt = x if dev else torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=self.device)
        if xt.dtype != torch.float64 or xt.shape != (self.n,):
            raise ShapeMismatchError(f"expected a float64 vector of length {self.n}, got {tuple(xt.shape)}")
        out = torch.empty_like(xt)
        self.apply_into(xt.contiguous(), out)
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
    log = {}
    errors = []

    def exchange(user, xp):
        try:
            x = xp.contents
            nsend, send_len = int(x.nsend), int(x.send_len)
            idx = np.ctypeslib.as_array(x.send_idx, shape=(nsend,)).copy() if nsend else np.zeros(0, np.int32)
            meta = (np.ctypeslib.as_array(x.send_meta, shape=(4 * nsend,)).reshape(-1, 4).copy() if nsend
                    else np.zeros((0, 4), np.int32))
            sizes = _sum_in_rank_order(_onehot(world, rank, (nsend, send_len)).ravel(),
                                       group, dev).reshape(world, 2).astype(np.int64)
            log.update(rank=rank, nblocks=int(x.nblocks), sent_blocks=nsend, sent_bytes=8 * send_len,
                       sent_meta=meta, per_rank=sizes.tolist())
            if rank == 0:
                for r in range(1, world):
                    nb, ln = int(sizes[r, 0]), int(sizes[r, 1])
                    if nb == 0:
                        continue
                    ridx = torch.empty(nb, dtype=torch.int32, device=dev)
                    rbuf = torch.empty(ln, dtype=torch.float64, device=dev)
                    _recv(ridx, r, group)
                    _recv(rbuf, r, group)
                    hidx = ridx.cpu().numpy()
                    N.order_after_torch(N.context(device), device)  # the receive has landed
                    N.raise_for(N.lib().sgf_exchange_accumulate(x.accum, hidx.ctypes.data, nb, rbuf.data_ptr()))
            elif nsend:
                _send(torch.as_tensor(idx, device=dev), 0, group)
                _send(_wrap(x.send_buf, send_len, dev), 0, group)
            return 0
        except Exception as e:  # surfaces as a factorize failure
            errors.append(e)
            return 1

    cb = N.EXCHANGE_FN(exchange)
    plan_info = {}

    def shard(hier, skip_levels, compression):
        cell_rank, stop, p = shard_plan(hier, world, skip_levels, compression)
        plan_info.update(stop=stop, partition_level=p, cell_rank=cell_rank)
        return {"rank": rank, "count": max(world, 2), "cell_rank": cell_rank, "stop_level": stop,
                "exchange": cb}

    try:
        pre = factorize(problem, device=device, _shard=shard, **kw)
    except Exception:
        if errors:
            raise errors[0]
        raise
    return ShardedPreconditioner(pre, group, dev, log, plan_info)


def _onehot(world, rank, vals):
    out = np.zeros((world, len(vals)))
    out[rank] = vals
    return out


# ---------------------------------------------------------------------------
# distributed PCG with halo exchange
# ---------------------------------------------------------------------------
class _HaloPlan:
    """Owned rows of A on this rank and the halo exchange its SpMV needs.
    Every rank derives every send list from the (replicated) pattern of A and
    the global ownership, so no request round is needed."""

    def __init__(self, A, precond):
        import torch

        dist = _dist()
        group, dev = precond.group, precond.device
        rank, world = precond.rank, precond.world
        n = A.shape[0]
        own = np.full(n, -1, np.int32)
        own[precond.owned] = rank
        t = torch.as_tensor(own.astype(np.int64))
        t = _comm(t.to(dev) if not _is_gloo(group) else t, group)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        owner = t.cpu().numpy().astype(np.int32)
        if (owner < 0).any():
            raise ValueError("sharded PCG: some unknowns have no owning rank")
        A = sp.csr_matrix(A)
        self.owner = owner
        rows_of = [np.flatnonzero(owner == r) for r in range(world)]
        # halo of rank s = columns its rows reference, owned by others
        self.send = {}   # peer -> indices this rank sends it (sorted, global ids)
        self.recv = {}   # peer -> indices this rank receives from it
        for s in range(world):
            cols = np.unique(A[rows_of[s]].indices) if rows_of[s].size else np.zeros(0, np.int64)
            halo = cols[owner[cols] != s]
            for r in np.unique(owner[halo]):
                ids = halo[owner[halo] == r]
                if r == rank and s != rank:
                    self.send[s] = ids
                if s == rank and r != rank:
                    self.recv[int(r)] = ids
        mask = np.zeros(n, bool)
        mask[rows_of[rank]] = True
        Aown = sp.diags(mask.astype(float)) @ A  # owned rows, others empty
        Aown = sp.csr_matrix(Aown)
        Aown.eliminate_zeros()
        # keep stored zeros of owned rows out of the picture only if A had none
        self.csr = DeviceCSR(Aown, device=dev.index)
        self.halo_bytes = 8 * sum(len(v) for v in self.recv.values())
        i32 = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int32), device=dev)  # noqa: E731
        self.send_idx = {k: i32(v) for k, v in self.send.items()}
        self.recv_idx = {k: i32(v) for k, v in self.recv.items()}
        self.send_buf = {k: torch.empty(len(v), dtype=torch.float64, device=dev) for k, v in self.send.items()}
        self.recv_buf = {k: torch.empty(len(v), dtype=torch.float64, device=dev) for k, v in self.recv.items()}
        self.vh = torch.empty(n, dtype=torch.float64, device=dev)
        self.n = n


_PLANS = {}


def pcg_sharded(A, b, precond, tol=1e-10, maxit=5000, true_residual_every=50):
    """Collective PCG (reference krylov.py:34-102) with a ShardedPreconditioner
    on distributed vectors (native sgf_pcg_dist).  A is the (host, scipy)
    matrix, replicated on every rank, or a DeviceCSR built from one
    (`DeviceCSR(A)`, whose host pattern is kept); b the same vector on every
    rank (numpy or a CUDA tensor).  Returns (x, SolveReport) on every rank."""
    import torch

    dist = _dist()
    Ah = A if sp.issparse(A) else getattr(A, "_host", None)
    if Ah is None:
        raise TypeError("pcg_sharded needs the host matrix (scipy) to plan the halo exchange")
    n = Ah.shape[0]
    if precond.n != n:
        raise ShapeMismatchError("preconditioner and matrix sizes differ")
    import hashlib

    # the ownership is the same for every factorization of one problem on one
    # process group: the plan (owned-row CSR, halo lists) is built once.
    # Building it is a collective, so hit or miss must come out the same on
    # every rank: the cached entry holds the matrix's arrays themselves and is
    # matched by object identity (never by id(), which a dead object's
    # successor can reuse on one rank and not on another).
    arrays = (Ah.indptr, Ah.indices, Ah.data)
    key = (precond.rank, precond.world, hashlib.blake2b(precond.owned.tobytes(), digest_size=16).hexdigest())
    ent = _PLANS.get("plan")
    if ent is not None and ent[0] == key and all(a is b_ for a, b_ in zip(ent[1], arrays)):
        plan = ent[2]
    else:
        _PLANS.clear()
        plan = _HaloPlan(Ah, precond)
        _PLANS["plan"] = (key, arrays, plan)
    dev = precond.device
    ctx = precond.pre._ctx
    L = N.lib()
    group = precond.group
    is_dev = not isinstance(b, np.ndarray) and getattr(b, "is_cuda", False)
    bt = b if is_dev else torch.as_tensor(np.ascontiguousarray(b, dtype=np.float64), device=dev)
    bm = precond.masked(bt.contiguous())
    x = torch.empty(n, dtype=torch.float64, device=dev)
    err = []

    def matvec(user, pin, pout):
        try:
            # vh = v with the halo entries other ranks own, then the owned-row SpMV
            N.raise_for(L.sgf_memcpy(ctx, plan.vh.data_ptr(), pin, 8 * n), ctx)
            for peer, idx in plan.send_idx.items():
                N.raise_for(L.sgf_vec_gather(ctx, pin, idx.data_ptr(), plan.send_buf[peer].data_ptr(), idx.numel()),
                            ctx)
            ops = []
            gloo = _is_gloo(group)
            sends = {p: _comm(t, group) for p, t in plan.send_buf.items()}
            recvs = {p: _comm(t, group) for p, t in plan.recv_buf.items()}
            for peer, t in sends.items():
                ops.append(dist.P2POp(dist.isend, t, peer, group))
            for peer, t in recvs.items():
                ops.append(dist.P2POp(dist.irecv, t, peer, group))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            if gloo:
                for peer in plan.recv_idx:
                    plan.recv_buf[peer].copy_(recvs[peer])
            N.order_after_torch(ctx, dev.index)  # the receives have landed
            for peer, idx in plan.recv_idx.items():
                N.raise_for(L.sgf_vec_scatter(ctx, plan.recv_buf[peer].data_ptr(), idx.data_ptr(),
                                              plan.vh.data_ptr(), idx.numel()), ctx)
            N.raise_for(L.sgf_spmv(plan.csr._h, plan.vh.data_ptr(), pout, 1), ctx)
            return 0
        except Exception as e:  # noqa: BLE001
            err.append(e)
            return N.SGF_CUDA

    def precondition(user, pin, pout):
        try:
            precond.apply_dist(pin, pout)
            return 0
        except Exception as e:  # noqa: BLE001
            err.append(e)
            return N.SGF_CUDA

    def reduce(user, vals, k):
        try:
            v = np.ctypeslib.as_array(vals, shape=(k,))
            v[:] = _sum_in_rank_order(v.copy(), group, dev)
            return 0
        except Exception as e:  # noqa: BLE001
            err.append(e)
            return 1

    fmv, fpc, fred = N.MATVEC_FN(matvec), N.PRECOND_FN(precondition), N.REDUCE_FN(reduce)
    rep = N.PcgReport()
    hist = np.zeros(maxit + 2)
    st = L.sgf_pcg_dist(ctx, n, fmv, None, fpc, None, fred, None, bm.data_ptr(), x.data_ptr(), float(tol),
                        int(maxit), int(true_residual_every), C.byref(rep), hist.ctypes.data)
    if err:
        raise err[0]
    N.raise_for(st, ctx)
    _allreduce_sum(x, group)  # owned pieces -> the whole solution on every rank
    report = SolveReport(iterations=rep.iterations, residual_history=hist[:rep.history_len].tolist(),
                         converged=bool(rep.converged), wall_time=rep.wall_time,
                         final_rel_residual=rep.final_rel_residual)
    return (x if is_dev else x.cpu().numpy()), report
