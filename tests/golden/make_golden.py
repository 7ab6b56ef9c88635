"""Generate golden fixtures by running the REFERENCE package itself.

Run once in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [--with-cfg2]
    python tests/golden/make_golden.py cfg4_full   # one slim full-size case
                                                   # (cfg3_full cfg4_full cfg5_full tpfa40_b9; ~15 min, ~49 GB each)

It imports `polyprec` read-only from /root/reference/pkg/src with the BLAS
pinned as SURVEY.md 8c prescribes (OPENBLAS_NUM_THREADS=1,
OPENBLAS_CORETYPE=Haswell), wraps `pivoted_qr` non-invasively to record each
compression's column permutation, and writes one compressed .npz per case
with the inputs, the hierarchy, the rank trace, the permutations, the stats,
apply_inverse / apply_operator of a seeded vector, the PCG history and (for
tiny cases) every factor's entries.  The GPU box has no /root/reference:
the fixtures are what travels.
"""

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_CORETYPE", "Haswell")

import json  # noqa: E402
import sys  # noqa: E402

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
import polyprec as pp  # noqa: E402
import polyprec.factorization as pfz  # noqa: E402
from polyprec import problems as pprob  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
KIND = {"cell0": 0, "cell1": 1, "cell2": 2, "cell3": 3, "general": 4}

_perms = []
_orig_qr = pfz.pivoted_qr


def _recording_qr(A, rank_tol=1e-10, full_q=False):
    out = _orig_qr(A, rank_tol=rank_tol, full_q=full_q)
    _perms.append(np.asarray(out.perm, dtype=np.int64))
    return out


pfz.pivoted_qr = _recording_qr


def poisson2d(n):
    h = 1.0 / (n + 1)
    T = pprob._tridiag_1d(n, h)
    I = sp.identity(n, format="csr")
    A = (sp.kron(I, T) + sp.kron(T, I)).tocsr()
    grid = pp.CartesianGrid(dims=(n, n, 1), spacing=(h, h, h))
    coords = pprob._lattice_coords((n, n, 1), (h, h, h), offset=1.0)
    return pp.ProblemInstance(matrix=A, coords=coords, grid=grid, components=1,
                              rhs=np.ones(n * n), label=f"p2d{n}")


def aniso(n, eps):
    h = 1.0 / (n + 1)
    T = pprob._tridiag_1d(n, h)
    I = sp.identity(n, format="csr")
    A = (sp.kron(I, sp.kron(I, T)) + sp.kron(I, sp.kron(T, I))
         + sp.kron(eps * T, sp.kron(I, I))).tocsr()
    grid = pp.CartesianGrid(dims=(n, n, n), spacing=(h, h, h))
    coords = pprob._lattice_coords((n, n, n), (h, h, h), offset=1.0)
    return pp.ProblemInstance(matrix=A, coords=coords, grid=grid, components=1,
                              rhs=np.ones(n ** 3), label=f"aniso{n}")


def tpfa(n, seed):
    """darcy_tpfa (x- Dirichlet) + the five other half-cell terms."""
    h = 1.0 / n
    a = 10.0 ** np.random.default_rng(seed).uniform(-3, 3, n ** 3)
    fld = pprob.ScalarField(dims=(n, n, n), values=a)
    prob = pprob.darcy_tpfa(fld, spacing=h, dirichlet_face="x-")
    lam = fld.cube()
    ids = np.arange(n ** 3).reshape((n, n, n), order="F")
    extra = np.zeros(n ** 3)
    geo = h * h / h
    for axis, side in ((0, -1), (1, 0), (1, -1), (2, 0), (2, -1)):
        s2 = [slice(None)] * 3
        s2[axis] = side
        np.add.at(extra, ids[tuple(s2)].ravel(), 2.0 * lam[tuple(s2)].ravel() * geo)
    A = (prob.matrix + sp.diags(extra)).tocsr()
    return pp.ProblemInstance(matrix=A, coords=prob.coords, grid=prob.grid, components=1,
                              rhs=np.zeros(n ** 3), label=f"tpfa{n}")


def elast(ne, seed):
    h = 1.0 / ne
    vx = ne + 1
    nv = vx ** 3
    E = 10.0 ** np.random.default_rng(seed).uniform(-1, 1, ne ** 3)
    nu = 0.3
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    K1 = pprob.hex_element_stiffness((h, h, h), 1.0, 0.0)
    K2 = pprob.hex_element_stiffness((h, h, h), 0.0, 1.0)
    e = np.arange(ne ** 3)
    ei, ej, ek = e % ne, (e // ne) % ne, e // (ne * ne)
    corners = np.empty((len(e), 8), dtype=np.int64)
    for c in range(8):
        cx, cy, cz = c & 1, (c >> 1) & 1, (c >> 2) & 1
        corners[:, c] = (ei + cx) + vx * ((ej + cy) + vx * (ek + cz))
    dofs = np.concatenate([corners + comp * nv for comp in range(3)], axis=1)
    data = lam[:, None, None] * K1 + mu[:, None, None] * K2
    K = sp.coo_matrix((data.ravel(), (np.repeat(dofs, 24, axis=1).ravel(),
                                      np.tile(dofs, (1, 24)).ravel())),
                      shape=(3 * nv, 3 * nv)).tocsr()
    vids = np.arange(nv)
    free_v = vids[vids % vx != 0]
    free = np.concatenate([free_v + c * nv for c in range(3)])
    A = K[free][:, free].tocsr()
    coords = pprob._lattice_coords((vx, vx, vx), (h, h, h), offset=0.0)[free_v]
    grid = pp.CartesianGrid(dims=(vx - 1, vx, vx), spacing=(h, h, h), components_per_vertex=3)
    return pp.ProblemInstance(matrix=A, coords=coords, grid=grid, components=3,
                              rhs=np.zeros(A.shape[0]), label=f"elast{ne}")


def hierarchy_arrays(prob, scheme, b):
    builder = pp.build_general_hierarchy if scheme == "gen-all-all" else pp.build_nested_hierarchy
    H = builder(prob.grid, b)
    out = {}
    for t, lev in enumerate(H.levels):
        cov = np.full(prob.grid.n_vertices, -1, dtype=np.int32)
        for c in lev.cells:
            cov[c.vertex_ids] = c.id
        out[f"h{t}_cov"] = cov
        out[f"h{t}_kind"] = np.array([KIND[c.kind] for c in lev.cells], dtype=np.int8)
        out[f"h{t}_interior"] = np.array([c.role == "interior" for c in lev.cells], dtype=np.int8)
        if lev.father:
            fa = np.full(len(lev.cells), -1, dtype=np.int32)
            for k, v in lev.father.items():
                fa[k] = v
            out[f"h{t}_father"] = fa
    out["h_levels"] = np.int64(len(H.levels))
    return out


def run_case(name, prob, opts, store_factors=False, pcg_tol=1e-12, rhs_seed=0, lowrank=False,
             slim=False):
    _perms.clear()
    P = pp.factorize(prob, **opts)
    perms = list(_perms)
    A = prob.matrix
    n = prob.n
    rhs = np.random.default_rng(rhs_seed).uniform(-1.0, 1.0, n)
    d = dict(
        indptr=A.indptr.astype(np.int64), indices=A.indices.astype(np.int64), data=A.data,
        coords=prob.coords, dims=np.array(prob.grid.dims), spacing=np.array(prob.grid.spacing),
        comps=np.int64(prob.components),
        opts=json.dumps(opts), stats=json.dumps(P.stats),
        rank_trace=np.array(P.rank_trace.entries, dtype=np.int64).reshape(-1, 3),
        perm_ptr=np.cumsum([0] + [len(p) for p in perms]).astype(np.int64),
        perm_all=np.concatenate(perms) if perms else np.zeros(0, np.int64),
        rhs=rhs, apply_inverse=P.apply_inverse(rhs), apply_operator=P.apply_operator(rhs),
        half_inverse=P.apply_half_inverse(rhs),
        blas=json.dumps({k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OPENBLAS_CORETYPE")}),
        versions=json.dumps({"numpy": np.__version__, "scipy": __import__("scipy").__version__,
                             "polyprec": pp.__version__}),
    )
    d.update(hierarchy_arrays(prob, opts.get("scheme", "nest-2-2"),
                              P.stats["b"]))
    if pcg_tol is not None:
        x, rep = pp.pcg(lambda v: A @ v, rhs, precond=P.apply_inverse, tol=pcg_tol, maxit=5000)
        d.update(pcg_x=x, pcg_hist=np.array(rep.residual_history), pcg_iters=np.int64(rep.iterations),
                 pcg_final=np.float64(rep.final_rel_residual), pcg_conv=np.int8(rep.converged))
    if store_factors:
        for k, f in enumerate(P.factors):
            typ = type(f).__name__
            d[f"f{k}_type"] = np.array(typ)
            d[f"f{k}_idx"] = f.idx.astype(np.int64)
            d[f"f{k}_L"] = f.L
            d[f"f{k}_node"] = np.int64(-1 if f.node is None else f.node)
            if typ == "EliminationFactor":
                d[f"f{k}_E"] = (np.vstack([E for _, E in f.couplings]) if f.couplings
                                else np.zeros((0, len(f.idx))))
                d[f"f{k}_Eidx"] = (np.concatenate([i for i, _ in f.couplings]).astype(np.int64)
                                   if f.couplings else np.zeros(0, np.int64))
            if typ == "CompressionFactor":
                d[f"f{k}_Q"] = f.Q
                d[f"f{k}_r"] = np.int64(f.retained)
        d["nfactors"] = np.int64(len(P.factors))
    if slim:
        # large config: the matrix is regenerated by the product's generator
        # (checked equal on the small cases); keep only the verdicts
        for k in [k for k in d if k.startswith("h") and k != "half_inverse"] + [
                "indptr", "indices", "data", "coords", "apply_operator", "half_inverse", "pcg_x"]:
            d.pop(k, None)
    if lowrank:
        _perms.clear()
        Pl = pp.factorize(prob, **dict(opts, mode="lowrank"), rank_trace=P.rank_trace)
        lp = list(_perms)
        d["lowrank_perm_ptr"] = np.cumsum([0] + [len(p) for p in lp]).astype(np.int64)
        d["lowrank_perm_all"] = np.concatenate(lp) if lp else np.zeros(0, np.int64)
        d["lowrank_apply_inverse"] = Pl.apply_inverse(rhs)
        d["lowrank_stats"] = json.dumps(Pl.stats)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **d)
    print(name, "n=%d" % n, "factors=%d" % len(P.factors), "ranks=%d" % len(P.rank_trace),
          "bytes=%d" % os.path.getsize(path), flush=True)


# ---------------------------------------------------------------------------
# Slim fixtures for the full-size BASELINE configs (cfg3/4/5) and the 40^3
# TPFA case whose level-3 node has >= 1024 unknowns (INT8-emulated products
# on the GPU).  Dense factors and n-vectors are far too large to commit, so a
# fixture keeps: digests of the matrix and of the hierarchy (bitwise pins of
# the product's generators and partition), the rank trace, every QR
# permutation (for pivot replay), the stats, strided samples and seeded
# Gaussian projections of apply_inverse / apply_operator / the PCG solution,
# the whole PCG history, and for a selection of factors (the emulated
# eliminations, the compressions after them, the final dense factor) their
# index sets, two columns and seeded projections of L / E / Q1.  Seeds:
# vector projections rng(7).standard_normal((4, n)); factor k uses
# rng(1000 + k) for the m-side and rng(2000 + k) for the c-side.
# ---------------------------------------------------------------------------

import hashlib  # noqa: E402

STRIDE = 32


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def matrix_digest(A):
    A = A.tocsr()
    A.sort_indices()
    return digest(A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data.astype(np.float64))


def hierarchy_digest(prob, scheme, b):
    arrs = hierarchy_arrays(prob, scheme, b)
    L = int(arrs["h_levels"])
    out = []
    for t in range(L):
        parts = [arrs[f"h{t}_cov"], arrs[f"h{t}_kind"], arrs[f"h{t}_interior"]]
        if f"h{t}_father" in arrs:
            parts.append(arrs[f"h{t}_father"].astype(np.int32))
        out.append(digest(*parts))
    return out


def vec_sample(d, key, y, proj):
    d[f"{key}_s"] = np.ascontiguousarray(y[::STRIDE])
    d[f"{key}_p"] = proj @ y
    d[f"{key}_norm"] = np.float64(np.linalg.norm(y))


def select_factors(P):
    kinds = [type(f).__name__ for f in P.factors]
    ms = [len(f.idx) for f in P.factors]
    pick = set()

    def spread(lst, k=3):
        if not lst:
            return []
        if len(lst) <= k:
            return lst
        return [lst[0], lst[len(lst) // 2], lst[-1]][:k]

    big = [k for k, (t, m) in enumerate(zip(kinds, ms)) if t == "EliminationFactor" and m >= 1024]
    mid = [k for k, (t, m) in enumerate(zip(kinds, ms)) if t == "EliminationFactor" and 640 <= m < 1024]
    small = [k for k, (t, m) in enumerate(zip(kinds, ms)) if t == "EliminationFactor" and m < 640]
    comp = [k for k, t in enumerate(kinds) if t == "CompressionFactor"]
    pick.update(spread(big))
    pick.update(spread(mid, 2))
    pick.update(small[:1])
    pick.update(spread(comp))
    pick.update(comp[-3:])
    pick.update(k for k, t in enumerate(kinds) if t == "DenseFactor")
    return sorted(pick)


def sample_factor(d, k, f):
    typ = type(f).__name__
    m = len(f.idx)
    W = np.random.default_rng(1000 + k).standard_normal((2, m))
    cols = np.random.default_rng(1000 + k).choice(m, size=min(2, m), replace=False) if m else np.zeros(0, int)
    d[f"f{k}_type"] = np.array(typ)
    d[f"f{k}_idx"] = f.idx.astype(np.int64)
    d[f"f{k}_node"] = np.int64(-1 if f.node is None else f.node)
    L = f.L
    d[f"f{k}_LW"] = L @ W.T
    d[f"f{k}_LtW"] = L.T @ W.T
    d[f"f{k}_Lcols"] = np.asarray(cols, np.int64)
    d[f"f{k}_Lcol"] = L[:, cols]
    if typ == "EliminationFactor":
        if f.couplings:
            E = np.vstack([E for _, E in f.couplings])
            Eidx = np.concatenate([i for i, _ in f.couplings]).astype(np.int64)
        else:
            E, Eidx = np.zeros((0, m)), np.zeros(0, np.int64)
        V = np.random.default_rng(2000 + k).standard_normal((2, len(Eidx)))
        d[f"f{k}_Eidx"] = Eidx
        d[f"f{k}_EW"] = E @ W.T
        d[f"f{k}_EtV"] = E.T @ V.T
        d[f"f{k}_Ecol"] = E[:, cols]
    if typ == "CompressionFactor":
        r = int(f.retained)
        Q1 = f.Q[:, :r]
        d[f"f{k}_r"] = np.int64(r)
        d[f"f{k}_Q1col"] = np.ascontiguousarray(Q1[:, :min(r, 4)])
        Wr = np.random.default_rng(3000 + k).standard_normal((2, r))
        d[f"f{k}_Q1W"] = Q1 @ Wr.T
        d[f"f{k}_Q1tW"] = Q1.T @ W.T


def run_full(name, prob, opts, rhs_seed, full_vectors=False):
    import time
    _perms.clear()
    A = prob.matrix.tocsr()
    n = prob.n
    t0 = time.perf_counter()
    P = pp.factorize(prob, **opts)
    t_f = time.perf_counter() - t0
    perms = list(_perms)
    rhs = np.random.default_rng(rhs_seed).uniform(-1.0, 1.0, n)
    proj = np.random.default_rng(7).standard_normal((4, n))
    d = dict(
        full=np.int8(1), n=np.int64(n), rhs_seed=np.int64(rhs_seed),
        matrix_digest=np.array(matrix_digest(A)),
        hier_digest=np.array(hierarchy_digest(prob, opts.get("scheme", "nest-2-2"), P.stats["b"])),
        opts=json.dumps(opts), stats=json.dumps(P.stats),
        rank_trace=np.array(P.rank_trace.entries, dtype=np.int64).reshape(-1, 3),
        perm_ptr=np.cumsum([0] + [len(p) for p in perms]).astype(np.int64),
        perm_all=np.concatenate(perms) if perms else np.zeros(0, np.int64),
        blas=json.dumps({k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OPENBLAS_CORETYPE")}),
        versions=json.dumps({"numpy": np.__version__, "scipy": __import__("scipy").__version__,
                             "polyprec": pp.__version__}),
    )
    y = P.apply_inverse(rhs)
    vec_sample(d, "apply_inverse", y, proj)
    if full_vectors:
        d["apply_inverse"] = y
    w = P.apply_operator(rhs)
    vec_sample(d, "apply_operator", w, proj)
    del y, w
    t0 = time.perf_counter()
    x, rep = pp.pcg(lambda v: A @ v, rhs, precond=P.apply_inverse, tol=1e-12, maxit=5000)
    t_s = time.perf_counter() - t0
    d.update(pcg_hist=np.array(rep.residual_history), pcg_iters=np.int64(rep.iterations),
             pcg_final=np.float64(rep.final_rel_residual), pcg_conv=np.int8(rep.converged))
    vec_sample(d, "pcg_x", x, proj)
    sel = select_factors(P)
    d["sampled_factors"] = np.array(sel, np.int64)
    d["nfactors"] = np.int64(len(P.factors))
    d["factor_types"] = np.array([{"EliminationFactor": 0, "CompressionFactor": 1, "DenseFactor": 2}[
        type(f).__name__] for f in P.factors], np.int8)
    d["factor_sizes"] = np.array([len(f.idx) for f in P.factors], np.int64)
    for k in sel:
        sample_factor(d, k, P.factors[k])
    d["ref_times"] = json.dumps({"t_factor_s": t_f, "t_solve_s": t_s, "host": os.uname().nodename,
                                 "cpus": os.cpu_count()})
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **d)
    print(name, "n=%d" % n, "factors=%d" % len(P.factors), "sampled=%d" % len(sel),
          "t_F=%.1f t_S=%.1f iters=%d" % (t_f, t_s, rep.iterations),
          "bytes=%d" % os.path.getsize(path), flush=True)


def augment_history_spread(name, prob, opts, rhs_seed):
    """Add the reference's own rounding sensitivity to a full-size fixture:
    the same factorization (pivots replayed from the fixture), then the PCG
    history once with the fixture's matvec `A @ v` (must reproduce the stored
    history bitwise) and once with `tril(A) @ v + triu(A, 1) @ v` (the same
    operator summed in another order: a rounding-level perturbation).  Ill-conditioned
    configs (cfg3, 10^6 contrast) amplify such perturbations through the CG
    recurrence far beyond 1e-10; pcg_hist_alt bounds what agreement with the
    reference can mean there."""
    path = os.path.join(HERE, f"{name}.npz")
    z = dict(np.load(path))
    A = prob.matrix.tocsr()
    n = prob.n
    rhs = np.random.default_rng(rhs_seed).uniform(-1.0, 1.0, n)
    P = pp.factorize(prob, **opts)
    x, rep = pp.pcg(lambda v: A @ v, rhs, precond=P.apply_inverse, tol=1e-12, maxit=5000)
    same = np.array_equal(np.array(rep.residual_history), z["pcg_hist"])
    import scipy.sparse as sps
    Al, Au = sps.tril(A).tocsr(), sps.triu(A, 1).tocsr()
    x2, rep2 = pp.pcg(lambda v: Al @ v + Au @ v, rhs, precond=P.apply_inverse, tol=1e-12, maxit=5000)
    z["pcg_hist_alt"] = np.array(rep2.residual_history)
    z["pcg_iters_alt"] = np.int64(rep2.iterations)
    z["pcg_hist_repro"] = np.int8(same)
    np.savez_compressed(path, **z)
    h, a = z["pcg_hist"], z["pcg_hist_alt"]
    k = min(len(h), len(a)) - 1
    print(name, "history reproduced bitwise:", same, "iters", rep.iterations, rep2.iterations,
          "max rel spread %.2e" % np.max(np.abs(h[:k] - a[:k]) / h[:k]), flush=True)


AUGMENT = {
    "cfg3_full": lambda: augment_history_spread("cfg3_full", tpfa(128, 2),
                                                dict(scheme="nest-2-2", degree=1, b=9, rank_tol=1e-2), 3),
    "cfg4_full": lambda: augment_history_spread("cfg4_full", aniso(128, 1e-3),
                                                dict(scheme="nest-2-2", degree=1, b=9, rank_tol=1e-3), 4),
    "cfg5_full": lambda: augment_history_spread("cfg5_full", elast(64, 5),
                                                dict(scheme="nest-2-2", degree=1, b=6, rank_tol=1e-2), 6),
    "tpfa40_b9": lambda: augment_history_spread("tpfa40_b9", tpfa(40, 2),
                                                dict(scheme="nest-2-2", degree=1, b=9, rank_tol=1e-2), 3),
}


FULL_CASES = {
    "cfg3_full": lambda: run_full("cfg3_full", tpfa(128, 2), dict(scheme="nest-2-2", degree=1, b=9, rank_tol=1e-2),
                                  rhs_seed=3),
    "cfg4_full": lambda: run_full("cfg4_full", aniso(128, 1e-3),
                                  dict(scheme="nest-2-2", degree=1, b=9, rank_tol=1e-3), rhs_seed=4),
    "cfg5_full": lambda: run_full("cfg5_full", elast(64, 5), dict(scheme="nest-2-2", degree=1, b=6, rank_tol=1e-2),
                                  rhs_seed=6),
    "tpfa40_b9": lambda: run_full("tpfa40_b9", tpfa(40, 2), dict(scheme="nest-2-2", degree=1, b=9, rank_tol=1e-2),
                                  rhs_seed=3, full_vectors=True),
}


def main():
    T = "nest-2-2"
    run_case("p3d9_exact", pp.poisson7(9), dict(scheme=T, degree=1, mode="exact"), store_factors=True)
    run_case("p3d12_b3", pp.poisson7(12), dict(scheme=T, degree=1, b=3, rank_tol=1e-2),
             store_factors=True)
    run_case("p3d10_deg2", pp.poisson7(10), dict(scheme=T, degree=2, rank_tol=1e-10, skip_levels=1),
             store_factors=True)
    run_case("p2d32_b5", poisson2d(32), dict(scheme=T, degree=1, b=5, rank_tol=1e-2),
             store_factors=True)
    run_case("aniso14", aniso(14, 1e-3), dict(scheme=T, degree=1, b=3, rank_tol=1e-3), rhs_seed=4)
    run_case("tpfa12", tpfa(12, 2), dict(scheme=T, degree=1, b=3, rank_tol=1e-2), rhs_seed=3)
    run_case("elast3", elast(3, 5), dict(scheme=T, degree=1, b=3, rank_tol=1e-2), rhs_seed=6,
             store_factors=True)
    run_case("elast6_b6", elast(6, 5), dict(scheme=T, degree=1, b=6, rank_tol=1e-2), rhs_seed=6)
    run_case("elast8", elast(8, 5), dict(scheme=T, degree=1, b=3, rank_tol=1e-2, skip_levels=1),
             rhs_seed=6)
    run_case("p3d10_nall", pp.poisson7(10), dict(scheme="nest-all-all", degree=1, skip_levels=1))
    run_case("p3d10_n2all", pp.poisson7(10), dict(scheme="nest-2-all", degree=0, skip_levels=1))
    run_case("p3d9_gen", pp.poisson7(9), dict(scheme="gen-all-all", degree=0), lowrank=True)
    run_case("p3d9_gen_d1", pp.poisson7(9), dict(scheme="gen-all-all", degree=1), store_factors=True)
    run_case("cfg1", poisson2d(128), dict(scheme=T, degree=1, b=9, rank_tol=1e-2), rhs_seed=0)
    run_case("p3d40_b9", pp.poisson7(40, spacing=1.0 / 41),
             dict(scheme=T, degree=1, b=9, rank_tol=1e-2), rhs_seed=1)
    if "--with-cfg2" in sys.argv:
        run_case("cfg2", pp.poisson7(64, spacing=1.0 / 65),
                 dict(scheme=T, degree=1, b=9, rank_tol=1e-2), rhs_seed=1, slim=True)


if __name__ == "__main__":
    if "--augment" in sys.argv:
        for a in sys.argv[1:]:
            if a in AUGMENT:
                AUGMENT[a]()
        sys.exit(0)
    full = [a for a in sys.argv[1:] if a in FULL_CASES]
    if full:
        for a in full:
            FULL_CASES[a]()
    else:
        main()
