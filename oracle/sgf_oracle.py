"""CPU ORACLE for the factorize -> apply -> PCG path.  TEST INFRASTRUCTURE ONLY.

Nothing in the product (`paper_1907_03406_b200/`) may import this module.
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs use it, and only as the checker (or the timed CPU
baseline), never as a code path of the GPU implementation.

This is an independent numpy restatement of the algorithm of the reference
package `polyprec` (arXiv 1907.03406, Alg. 4.1).  Every function cites the
reference lines (paths relative to /root/reference/pkg/src/polyprec/) whose
behaviour it restates.  It is pinned against golden vectors produced by the
reference itself (`tests/golden/make_golden.py` -> `tests/golden/*.npz`,
checked by `tests/test_oracle_golden.py`).

Extras over the reference, both needed by the parity protocol (SURVEY.md
section 8c): every pivoted QR records its column permutation, and a run can
replay a recorded list of permutations so that rounding-level pivot near-ties
resolve the same way as in another implementation.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import solve_triangular

EPS = float(np.finfo(float).eps)
CHOL_RTOL = 1e-14            # densela.py:18
RANK_TOL_DEFAULT = 1e-10     # densela.py:21

SCHEMES = ("nest-all-all", "nest-2-all", "nest-2-2", "gen-all-all")   # factorization.py:32
COMPRESSED = {                                                        # factorization.py:37-42
    "nest-all-all": {"cell1", "cell2"},
    "nest-2-all": {"cell2"},
    "nest-2-2": {"cell2"},
    "gen-all-all": {"general"},
}
RAW_COUPLED = {"nest-2-2": {"cell0", "cell1"}}                        # factorization.py:47


class OracleNotSPD(ArithmeticError):
    """Cholesky breakdown (densela.py:106-110)."""


class OracleIndefinite(ArithmeticError):
    """Non-positive curvature in PCG (krylov.py:62-63, 71-72, 90-91)."""


# ---------------------------------------------------------------------------
# flop tally (densela.py:24-40; per-kernel formulas at :83, :115, :136, :141,
# :205).  Kept as a plain counter object owned by one factorization run.
# ---------------------------------------------------------------------------

class Tally:
    def __init__(self):
        self.flops = 0

    def __iadd__(self, v):
        self.flops += int(v)
        return self


# ---------------------------------------------------------------------------
# Partition hierarchy (partition.py:105-242).  Restated with the same
# lexicographic cell numbering: cell id = rank of the per-vertex label tuple
# (sep_x, grp_x, sep_y, grp_y, sep_z, grp_z).
# ---------------------------------------------------------------------------

def _labels(n, d, nested):
    i = np.arange(n)
    if not nested:                                   # partition.py:122-124
        return np.zeros(n, dtype=np.int64), i // d
    on_plane = ((i + 1) % d) == 0                    # partition.py:105-111
    grp = np.where(on_plane, (i + 1) // d - 1, i // d)
    return on_plane.astype(np.int64), grp


def _up_label(s, g, nested):
    """partition.py:114-119 (nested) and :126-127 (general)."""
    if nested and s:
        return (1, (g - 1) // 2) if g % 2 == 1 else (0, g // 2)
    return (0, g // 2)


@dataclass
class OLevel:
    vertices: list          # per cell: sorted vertex ids
    kinds: list             # per cell: "cell0".."cell3" or "general"
    roles: list             # per cell: "interior" / "separator"
    father: dict = field(default_factory=dict)


def hierarchy(dims, b, nested=True):
    """Levels of the nested (partition.py:202-217) or general (:220-229)
    family, built exactly as partition.py:179-199 does: period d doubles
    per level until a single cell remains."""
    nx, ny, nz = dims
    vid = np.arange(nx * ny * nz)
    ax_idx = (vid % nx, (vid // nx) % ny, vid // (nx * ny))
    levels, prev_map, d = [], None, b
    while True:
        labs = [_labels(n, d, nested) for n in dims]
        key = np.column_stack([np.column_stack((labs[a][0][ax_idx[a]], labs[a][1][ax_idx[a]]))
                               for a in range(3)])
        order = np.lexsort(key.T[::-1])
        ks = key[order]
        cut = np.flatnonzero(np.any(ks[1:] != ks[:-1], axis=1)) + 1
        bounds = np.concatenate(([0], cut, [len(order)]))
        verts, kinds, roles, tmap = [], [], [], {}
        for c in range(len(bounds) - 1):
            lab = tuple(int(v) for v in ks[bounds[c]])
            verts.append(np.sort(vid[order[bounds[c]:bounds[c + 1]]]))
            if nested:                                        # partition.py:131-135
                thick = 3 - (lab[0] + lab[2] + lab[4])
                kinds.append("cell%d" % thick)
                roles.append("interior" if thick == 3 else "separator")
            else:
                kinds.append("general")
                roles.append("separator")
            tmap[lab] = c
        levels.append(OLevel(verts, kinds, roles))
        if prev_map is not None:
            fa = {}
            for lab, c in prev_map.items():
                up = ()
                for a in range(3):
                    up += _up_label(lab[2 * a], lab[2 * a + 1], nested)
                fa[c] = tmap[up]
            levels[-2].father = fa
        if len(verts) == 1:
            return levels
        prev_map = tmap
        d *= 2


def cell_unknowns(verts, n_vertices, comps):
    """partition.py:232-242: component-major unknown ids."""
    if comps == 1:
        return verts.copy()
    return np.concatenate([verts + c * n_vertices for c in range(comps)])


def poly_basis(coords, degree, comps):
    """basis.py:27-62: monomials up to `degree`, block diagonal per
    component, columns scaled to unit max-norm (zero columns untouched)."""
    x, y, z = (np.asarray(coords, dtype=float)[:, a] for a in range(3))
    cols = [np.ones_like(x)]
    if degree >= 1:
        cols += [x, y, z]
    if degree >= 2:
        cols += [x * x, y * y, z * z, x * y, y * z, z * x]
    P = np.column_stack(cols)
    nv, ps = P.shape
    Pi = np.zeros((comps * nv, comps * ps))
    for c in range(comps):
        Pi[c * nv:(c + 1) * nv, c * ps:(c + 1) * ps] = P
    s = np.abs(Pi).max(axis=0)
    s[s == 0] = 1.0
    return Pi / s


# ---------------------------------------------------------------------------
# Dense kernels (densela.py:79-217)
# ---------------------------------------------------------------------------

def chol_lower(A, tally):
    """densela.py:87-116 -- left-looking column Cholesky with the relative
    pivot floor CHOL_RTOL * max(diag)."""
    A = np.asarray(A, dtype=float)
    m = A.shape[0]
    if not np.isfinite(A).all():
        raise ValueError("non-finite block")
    if m:
        big = np.abs(A).max()
        if big > 0 and np.abs(A - A.T).max() > 1e-12 * big:
            raise ValueError("block not symmetric")
    L = np.zeros_like(A)
    floor = CHOL_RTOL * max(A.diagonal().max(initial=0.0), 0.0)
    for j in range(m):
        row = L[j, :j]
        piv = A[j, j] - row @ row
        if not (piv > floor) or not np.isfinite(piv):
            raise OracleNotSPD("pivot %.3e at %d" % (piv, j))
        piv = np.sqrt(piv)
        L[j, j] = piv
        if j + 1 < m:
            L[j + 1:, j] = (A[j + 1:, j] - L[j + 1:, :j] @ row) / piv
    tally += m ** 3 // 3
    return L


def lsolve(L, B, tally):
    """densela.py:119-146 mode 'left': L^{-1} B."""
    tally += L.shape[0] ** 2 * B.shape[1]
    return solve_triangular(L, B, lower=True)


def rsolve_t(L, B, tally):
    """densela.py:137-141 mode 'right_t': B L^{-T}."""
    tally += L.shape[0] ** 2 * B.shape[0]
    return solve_triangular(L, B.T, lower=True).T


def mm(a, b, tally):
    """densela.py:79-84."""
    tally += 2 * a.shape[0] * a.shape[1] * b.shape[1]
    return a @ b


@dataclass
class QRCP:
    Q: np.ndarray
    R: np.ndarray
    perm: np.ndarray
    rank: int
    steps: int


def qrcp(A, tol, tally, replay=None):
    """densela.py:149-217 -- Householder QR with column-norm pivoting:
    first-argmax pivot on downdated squared norms, norm recomputation once a
    downdate lost half the digits (norm^2 <= eps * ref^2), early exit on
    numerically zero columns, full m-by-m Q, rank = #{|R_ii| > tol |R_00|}.

    replay: optional permutation recorded from another run; step k then
    pivots on the column whose original index is replay[k] (parity mode).
    """
    A = np.asarray(A, dtype=float)
    m, c = A.shape
    kmax = min(m, c)
    R = A.copy()
    perm = np.arange(c)
    V = np.zeros((m, kmax))
    tau = np.zeros(kmax)
    nrm2 = np.einsum("ij,ij->j", R, R)
    ref2 = nrm2.copy()
    floor = EPS * max(np.abs(A).max(initial=0.0), 1.0)
    steps = 0
    for k in range(kmax):
        if replay is not None and k < len(replay):
            p = int(np.flatnonzero(perm == replay[k])[0])
        else:
            p = k + int(np.argmax(nrm2[k:]))
        if nrm2[p] <= floor * floor:
            R[k:, k:] = 0.0
            break
        if p != k:
            for arr in (perm, nrm2, ref2):
                arr[[k, p]] = arr[[p, k]]
            R[:, [k, p]] = R[:, [p, k]]
        x = R[k:, k]
        xn = np.linalg.norm(x)
        if xn <= floor:
            R[k:, k:] = 0.0
            break
        sgn = -np.sign(x[0]) if x[0] != 0 else -1.0
        u1 = x[0] - sgn * xn
        v = x / u1
        v[0] = 1.0
        t = -sgn * u1 / xn
        R[k:, k:] -= np.outer(t * v, v @ R[k:, k:])
        R[k, k] = sgn * xn
        R[k + 1:, k] = 0.0
        V[k:, k] = v
        tau[k] = t
        steps = k + 1
        if k + 1 < c:
            nrm2[k + 1:] = np.maximum(nrm2[k + 1:] - R[k, k + 1:] ** 2, 0.0)
            stale = np.flatnonzero(nrm2[k + 1:] <= EPS * ref2[k + 1:]) + k + 1
            if stale.size:
                fresh = np.einsum("ij,ij->j", R[k + 1:, stale], R[k + 1:, stale])
                nrm2[stale] = fresh
                ref2[stale] = np.maximum(fresh, floor * floor)
    tally += 2 * m * c * c
    Q = np.eye(m)
    for k in range(steps - 1, -1, -1):
        v = V[k:, k]
        Q[k:, :] -= np.outer(tau[k] * v, v @ Q[k:, :])
    R = np.triu(R[:kmax, :])
    dg = np.abs(np.diagonal(R))
    rank = 0 if (dg.size == 0 or dg[0] == 0.0) else int((dg > tol * dg[0]).sum())
    return QRCP(Q, R, perm, rank, steps)


# ---------------------------------------------------------------------------
# Symmetric block storage (blockmatrix.py:14-170): blocks keyed (i, j), i<=j.
# ---------------------------------------------------------------------------

class Blocks:
    def __init__(self, sizes):
        self.size = dict(sizes)
        self.blk = {}
        self.adj = {i: set() for i in self.size}
        self.live = 0
        self.peak = 0

    def _put(self, key, arr):
        old = self.blk.get(key)
        if old is not None:
            self.live -= old.nbytes
        self.blk[key] = arr
        self.live += arr.nbytes
        self.peak = max(self.peak, self.live)
        if key[0] != key[1]:
            self.adj[key[0]].add(key[1])
            self.adj[key[1]].add(key[0])

    def has(self, i, j):
        return (min(i, j), max(i, j)) in self.blk

    def get(self, i, j):
        a = self.blk[(min(i, j), max(i, j))]
        return a if i <= j else a.T

    def put(self, i, j, a):
        a = np.asarray(a, dtype=float)
        assert a.shape == (self.size[i], self.size[j])
        if i > j:
            i, j, a = j, i, a.T
        self._put((i, j), a)

    def sub(self, i, j, d):
        """blockmatrix.py:65-72: blocks[key] += -d, creating zero fill."""
        if i > j:
            i, j, d = j, i, d.T
        if (i, j) not in self.blk:
            self._put((i, j), np.zeros((self.size[i], self.size[j])))
        self.blk[(i, j)] += -d

    def nbrs(self, i):
        return sorted(self.adj[i])

    def drop(self, i):
        for j in list(self.adj[i]):
            key = (min(i, j), max(i, j))
            self.live -= self.blk.pop(key).nbytes
            self.adj[j].discard(i)
        self.adj[i] = set()
        if (i, i) in self.blk:
            self.live -= self.blk.pop((i, i)).nbytes

    @classmethod
    def from_csr(cls, A, cell_idx):
        """blockmatrix.py:97-144 (entrywise scatter of a symmetric CSR)."""
        A = A.tocsr()
        n = A.shape[0]
        d = abs(A - A.T)
        big = abs(A).max() if A.nnz else 0.0
        if d.nnz and d.max() > 1e-12 * max(big, 1e-300):
            raise ValueError("matrix not symmetric")
        owner = np.full(n, -1, dtype=np.int64)
        loc = np.zeros(n, dtype=np.int64)
        for c, idx in cell_idx.items():
            owner[idx] = c
            loc[idx] = np.arange(len(idx))
        if (owner < 0).any():
            raise ValueError("cells do not cover the unknowns")
        M = cls({c: len(idx) for c, idx in cell_idx.items()})
        coo = A.tocoo()
        r, s = coo.row, coo.col
        lo = owner[r] > owner[s]
        bi = np.where(lo, owner[s], owner[r])
        bj = np.where(lo, owner[r], owner[s])
        li = np.where(lo, loc[s], loc[r])
        lj = np.where(lo, loc[r], loc[s])
        o = np.lexsort((bj, bi))
        bi, bj, li, lj, val = bi[o], bj[o], li[o], lj[o], coo.data[o]
        brk = np.flatnonzero((bi[1:] != bi[:-1]) | (bj[1:] != bj[:-1])) + 1
        st = np.concatenate(([0], brk))
        en = np.concatenate((brk, [len(val)]))
        for a, e in zip(st, en):
            i, j = int(bi[a]), int(bj[a])
            blk = np.zeros((M.size[i], M.size[j]))
            blk[li[a:e], lj[a:e]] = val[a:e]
            M._put((i, j), blk)
        return M


# ---------------------------------------------------------------------------
# Factors (factorization.py:112-213)
# ---------------------------------------------------------------------------

class OElim:
    kind = "elim"

    def __init__(self, node, idx, L, cpl):
        self.node, self.idx, self.L = node, np.asarray(idx), L
        self.couplings = cpl                    # [(idx_nb, E_nb)]
        self.Linv = solve_triangular(L, np.eye(len(L)), lower=True)

    def fwd(self, x):
        z = self.Linv @ x[self.idx]
        x[self.idx] = z
        for ii, E in self.couplings:
            x[ii] -= E @ z

    def bwd(self, x):
        acc = x[self.idx].copy()
        for ii, E in self.couplings:
            acc -= E.T @ x[ii]
        x[self.idx] = self.Linv.T @ acc

    def mul_t(self, x):
        acc = self.L.T @ x[self.idx]
        for ii, E in self.couplings:
            acc += E.T @ x[ii]
        x[self.idx] = acc

    def mul_f(self, x):
        xb = x[self.idx].copy()
        for ii, E in self.couplings:
            x[ii] += E @ xb
        x[self.idx] = self.L @ xb

    def apply_flops(self):
        m = len(self.idx)
        return 4 * m * m + 4 * m * sum(len(i) for i, _ in self.couplings)


class OComp:
    kind = "comp"

    def __init__(self, node, idx, L, Q, r, perm):
        self.node, self.idx, self.L, self.Q, self.retained = node, np.asarray(idx), L, Q, r
        self.perm = perm
        self.LQ = L @ Q
        self.inv = Q.T @ solve_triangular(L, np.eye(len(L)), lower=True)

    def fwd(self, x):
        x[self.idx] = self.inv @ x[self.idx]

    def bwd(self, x):
        x[self.idx] = self.inv.T @ x[self.idx]

    def mul_t(self, x):
        x[self.idx] = self.LQ.T @ x[self.idx]

    def mul_f(self, x):
        x[self.idx] = self.LQ @ x[self.idx]

    def apply_flops(self):
        return 4 * len(self.idx) ** 2


class ODense:
    kind = "dense"

    def __init__(self, idx, L):
        self.node, self.idx, self.L = None, np.asarray(idx), L
        self.Linv = solve_triangular(L, np.eye(len(L)), lower=True)

    def fwd(self, x):
        x[self.idx] = self.Linv @ x[self.idx]

    def bwd(self, x):
        x[self.idx] = self.Linv.T @ x[self.idx]

    def mul_t(self, x):
        x[self.idx] = self.L.T @ x[self.idx]

    def mul_f(self, x):
        x[self.idx] = self.L @ x[self.idx]

    def apply_flops(self):
        return 4 * len(self.idx) ** 2


@dataclass
class OPrecond:
    n: int
    factors: list
    stats: dict
    rank_trace: list          # [(level, node, rank)]
    perms: list               # one permutation per compression, in order
    Pi: np.ndarray
    levels: list = None       # the hierarchy used

    def apply_inverse(self, x):
        """factorization.py:255-262."""
        y = np.array(x, dtype=float, copy=True)
        for f in self.factors:
            f.fwd(y)
        for f in reversed(self.factors):
            f.bwd(y)
        return y

    def apply_operator(self, x):
        """factorization.py:264-271."""
        y = np.array(x, dtype=float, copy=True)
        for f in self.factors:
            f.mul_t(y)
        for f in reversed(self.factors):
            f.mul_f(y)
        return y

    def half_inverse(self, x):
        y = np.array(x, dtype=float, copy=True)
        for f in self.factors:
            f.fwd(y)
        return y


# ---------------------------------------------------------------------------
# Node operations (factorization.py:277-407)
# ---------------------------------------------------------------------------

@dataclass
class ONode:
    active: np.ndarray
    phi: np.ndarray
    role: str
    kind: str


def _eliminate(M, nodes, b, tally):
    """factorization.py:277-299."""
    L = chol_lower(M.get(b, b), tally)
    nb = M.nbrs(b)
    E = {j: rsolve_t(L, M.get(j, b), tally) for j in nb}
    cpl = [(nodes[j].active.copy(), E[j]) for j in nb]
    for p, i in enumerate(nb):
        for j in nb[p:]:
            u = mm(E[i], E[j].T, tally)
            if i == j:
                u = 0.5 * (u + u.T)
            M.sub(i, j, u)
    M.drop(b)
    M.size[b] = 0
    f = OElim(b, nodes[b].active, L, cpl)
    nodes[b].active = nodes[b].active[:0]
    nodes[b].phi = nodes[b].phi[:0]
    return f


def _compress(M, nodes, b, tol, raw_kinds, tally, mode="polynomial", forced=None,
              replay=None):
    """factorization.py:302-353."""
    nd = nodes[b]
    m = len(nd.active)
    L = chol_lower(M.get(b, b), tally)
    nb = M.nbrs(b)
    Mh = {j: lsolve(L, M.get(b, j), tally) for j in nb}
    LtPhi = mm(L.T, nd.phi, tally)
    if mode == "polynomial":
        cols = [LtPhi]
        for j in nb:
            cols.append(Mh[j] if nodes[j].kind in raw_kinds else mm(Mh[j], nodes[j].phi, tally))
        qr = qrcp(np.hstack(cols), tol, tally, replay)
        r = qr.rank
    else:
        Nm = np.hstack([Mh[j] for j in nb]) if nb else np.zeros((m, 0))
        qr = qrcp(Nm, tol, tally, replay)
        r = min(int(forced), m)
    Q1 = qr.Q[:, :r]
    f = OComp(b, nd.active, L, qr.Q, r, qr.perm)
    newc = {j: mm(Q1.T, Mh[j], tally) for j in nb}
    M.drop(b)
    M.size[b] = r
    if r > 0:
        M.put(b, b, np.eye(r))
        for j in nb:
            M.put(b, j, newc[j])
    nd.phi = mm(Q1.T, LtPhi, tally)
    nd.active = nd.active[:r]
    return f


def _merge(M, nodes, father, lev_next, pi):
    """factorization.py:356-407."""
    kids = {}
    for c, f in father.items():
        kids.setdefault(f, []).append(c)
    new_nodes, sizes, where = {}, {}, {}
    for fid in range(len(lev_next.vertices)):
        ch = sorted(kids.get(fid, []))
        pos = 0
        for c in ch:
            where[c] = (fid, pos)
            pos += len(nodes[c].active)
        act = np.concatenate([nodes[c].active for c in ch]) if ch else np.empty(0, np.int64)
        ph = np.vstack([nodes[c].phi for c in ch]) if ch else np.zeros((0, pi))
        new_nodes[fid] = ONode(act, ph, lev_next.roles[fid], lev_next.kinds[fid])
        sizes[fid] = pos
    N = Blocks(sizes)
    for (a, b) in sorted(M.blk):
        blk = M.blk[(a, b)]
        if blk.size == 0:
            continue
        fa, oa = where[a]
        fb, ob = where[b]
        ra, cb = blk.shape
        if not N.has(fa, fb):
            N.put(fa, fb, np.zeros((sizes[fa], sizes[fb])))
        if fa == fb:
            T = N.get(fa, fa)
            T[oa:oa + ra, ob:ob + cb] = blk
            if a != b:
                T[ob:ob + cb, oa:oa + ra] = blk.T
        elif fa < fb:
            N.get(fa, fb)[oa:oa + ra, ob:ob + cb] = blk
        else:
            N.get(fb, fa)[ob:ob + cb, oa:oa + ra] = blk.T
    return N, new_nodes


def factorize(A, coords, dims, comps=1, scheme="nest-2-2", degree=1, b=None,
              skip_levels=None, compression=True, mode="polynomial",
              rank_tol=RANK_TOL_DEFAULT, rank_trace=None, replay_perms=None):
    """factorization.py:410-573 (Alg. 4.1).  Returns OPrecond."""
    if scheme not in SCHEMES:
        raise ValueError(scheme)
    if mode == "exact":
        compression = False
    if mode == "lowrank" and compression and rank_trace is None:
        raise ValueError("lowrank needs a rank trace")
    nested = scheme != "gen-all-all"
    if b is None:
        b = 3 + degree if not nested else 3                       # :50-53
    if skip_levels is None:
        skip_levels = 0 if not nested else 2                      # :56-58
    nv = int(np.prod(dims))
    n = nv * comps
    levels = hierarchy(dims, b, nested)
    Pi = poly_basis(coords, degree, comps)
    nodes, cidx = {}, {}
    lev0 = levels[0]
    for c, verts in enumerate(lev0.vertices):
        idx = cell_unknowns(verts, nv, comps)
        cidx[c] = idx
        nodes[c] = ONode(idx.copy(), Pi[idx].copy(), lev0.roles[c], lev0.kinds[c])
    M = Blocks.from_csr(A, cidx)
    tally = Tally()
    factors, trace, perms = [], [], []
    replay_iter = iter(replay_perms) if replay_perms is not None else None
    rt_iter = iter(rank_trace) if rank_trace is not None else None
    comp_kinds = COMPRESSED[scheme]
    raw_kinds = RAW_COUPLED.get(scheme, set())
    max_seen = max_after = peak = 0
    per_level = []
    for t, lev in enumerate(levels):
        remaining = sum(len(v.active) for v in nodes.values())
        if remaining == 0 or (t > 0 and remaining < max_seen) or len(lev.vertices) == 1:
            break
        max_seen = max(max_seen, max(len(v.active) for v in nodes.values()))
        st = {"level": t + 1, "nodes": len(lev.vertices), "eliminated": 0,
              "compressed": 0, "ranks": []}
        for c in sorted(nodes):
            if nodes[c].role == "interior" and len(nodes[c].active):
                factors.append(_eliminate(M, nodes, c, tally))
                st["eliminated"] += 1
        if compression and t + 1 > skip_levels:
            for c in sorted(nodes):
                if nodes[c].kind not in comp_kinds or not len(nodes[c].active):
                    continue
                forced = None
                if mode == "lowrank":
                    try:
                        lv, rc, forced = next(rt_iter)
                    except StopIteration:
                        raise RuntimeError("rank trace exhausted")
                    if (lv, rc) != (t + 1, c):
                        raise RuntimeError("rank trace divergence")
                rp = next(replay_iter) if replay_iter is not None else None
                f = _compress(M, nodes, c, rank_tol, raw_kinds, tally,
                              mode="lowrank" if mode == "lowrank" else "polynomial",
                              forced=forced, replay=rp)
                factors.append(f)
                perms.append(f.perm)
                trace.append((t + 1, c, f.retained))
                st["ranks"].append(f.retained)
                st["compressed"] += 1
        sz = [len(v.active) for v in nodes.values()]
        if sz:
            max_after = max(max_after, max(sz))
        per_level.append(st)
        peak = max(peak, M.peak)
        if t + 1 < len(levels):
            old = M.live
            M, nodes = _merge(M, nodes, lev.father, levels[t + 1], Pi.shape[1])
            peak = max(peak, old + M.live)
        else:
            break
    rem = [c for c in sorted(nodes) if len(nodes[c].active)]
    if rem:
        off, pos = {}, 0
        for c in rem:
            off[c] = pos
            pos += M.size[c]
        D = np.zeros((pos, pos))
        for (a, bb), blk in M.blk.items():
            if a in off and bb in off:
                D[off[a]:off[a] + M.size[a], off[bb]:off[bb] + M.size[bb]] = blk
                if a != bb:
                    D[off[bb]:off[bb] + M.size[bb], off[a]:off[a] + M.size[a]] = blk.T
        Lf = chol_lower(D, tally)
        factors.append(ODense(np.concatenate([nodes[c].active for c in rem]), Lf))
        peak = max(peak, M.peak)
    if rt_iter is not None and list(rt_iter):
        raise RuntimeError("rank trace has unreplayed entries")
    stats = {
        "n": n, "scheme": scheme, "degree": degree,
        "mode": mode if compression else "exact", "b": b, "skip_levels": skip_levels,
        "levels": len(per_level), "per_level": per_level,
        "max_node_size": max_after, "max_node_seen": max_seen,
        "final_dense_size": len(factors[-1].idx) if rem else 0,
        "flops_factorize": tally.flops,
        "flops_apply": sum(f.apply_flops() for f in factors),
        "peak_blocks_bytes": peak, "factors": len(factors),
    }
    return OPrecond(n, factors, stats, trace, perms, Pi, levels)


# ---------------------------------------------------------------------------
# PCG (krylov.py:34-102)
# ---------------------------------------------------------------------------

@dataclass
class OReport:
    iterations: int
    residual_history: list
    converged: bool
    wall_time: float
    final_rel_residual: float


def pcg(Aop, b, M=None, tol=1e-10, maxit=5000, true_every=50):
    A = Aop if callable(Aop) else (lambda v: Aop @ v)
    P = M if M is not None else (lambda v: v)
    if M is not None and not callable(M):
        P = lambda v: M @ v  # noqa: E731
    b = np.asarray(b, dtype=float)
    t0 = time.perf_counter()
    bn = np.linalg.norm(b)
    if bn == 0.0:
        return np.zeros_like(b), OReport(0, [0.0], True, time.perf_counter() - t0, 0.0)
    x = np.zeros_like(b)
    r = b.copy()
    hist = [1.0]
    z = P(r)
    rz = float(r @ z)
    if rz <= 0.0:
        raise OracleIndefinite("r'Mr")
    p = z.copy()
    done = False
    it = 0
    while it < maxit:
        it += 1
        q = A(p)
        pq = float(p @ q)
        if pq <= 0.0:
            raise OracleIndefinite("p'Ap")
        al = rz / pq
        x += al * p
        r -= al * q
        if it % true_every == 0:
            r = b - A(x)
        rel = np.linalg.norm(r) / bn
        if rel <= tol:
            r = b - A(x)
            rel = np.linalg.norm(r) / bn
            hist.append(rel)
            if rel <= tol:
                done = True
                break
        else:
            hist.append(rel)
        z = P(r)
        rz2 = float(r @ z)
        if rz2 <= 0.0:
            raise OracleIndefinite("r'Mr")
        p = z + (rz2 / rz) * p
        rz = rz2
    fin = float(np.linalg.norm(b - A(x)) / bn)
    return x, OReport(it, hist, done and fin <= tol, time.perf_counter() - t0, fin)


def rank_trace_json(trace):
    """factorization.py:88-89 format."""
    return json.dumps({"entries": [list(e) for e in trace]})
