"""Run the REFERENCE package itself (oracle/_ref, built by oracle/build_ref.sh)
on one BASELINE config, timed the way the reference's own harness times it
(reference bench.py:157-166: t_F around `factorize`, t_S around
`pcg(lambda v: A @ v, rhs, precond=P.apply_inverse, tol=1e-12)`).

Baseline infrastructure only: bench.py's `--impl reference` arm and its
`cpu_baseline` leg run this as a subprocess (so the BLAS thread count is
fixed before numpy loads); nothing in the product imports it.

    OPENBLAS_NUM_THREADS=1 python oracle/ref_bench.py --cfg 4 [--n 40]

prints one JSON line {"t_factor_s", "t_solve_s", "iterations", ...}.  The
problems are built with the reference's own generators and containers
(`_tridiag_1d`, `_lattice_coords`, `darcy_tpfa`, `hex_element_stiffness`,
`CartesianGrid`, `ProblemInstance`) following SURVEY.md 8(d); the product's
generators reproduce these matrices bit for bit (tests/test_full_size_golden.py).
"""

import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


def load_reference():
    if not os.path.isdir(os.path.join(REF, "polyprec")):
        raise SystemExit(f"oracle/_ref is missing: run oracle/build_ref.sh (build())")
    sys.path.insert(0, REF)
    import polyprec

    return polyprec


def build(pp, cfg, n=None):
    """(ProblemInstance, b, rank_tol, rhs seed) for BASELINE config `cfg`,
    optionally at a smaller grid size n."""
    import numpy as np
    import scipy.sparse as sp
    from polyprec import problems as pprob

    if cfg == 1:
        n = n or 128
        h = 1.0 / (n + 1)
        T = pprob._tridiag_1d(n, h)
        I = sp.identity(n, format="csr")
        A = (sp.kron(I, T) + sp.kron(T, I)).tocsr()
        grid = pp.CartesianGrid(dims=(n, n, 1), spacing=(h, h, h))
        coords = pprob._lattice_coords((n, n, 1), (h, h, h), offset=1.0)
        return pp.ProblemInstance(matrix=A, coords=coords, grid=grid, components=1, rhs=np.zeros(n * n),
                                  label="cfg1"), 9, 1e-2, 0
    if cfg == 2:
        n = n or 64
        return pp.poisson7(n, spacing=1.0 / (n + 1)), 9, 1e-2, 1
    if cfg == 4:
        n = n or 128
        h = 1.0 / (n + 1)
        T = pprob._tridiag_1d(n, h)
        I = sp.identity(n, format="csr")
        A = (sp.kron(I, sp.kron(I, T)) + sp.kron(I, sp.kron(T, I)) + sp.kron(1e-3 * T, sp.kron(I, I))).tocsr()
        grid = pp.CartesianGrid(dims=(n, n, n), spacing=(h, h, h))
        coords = pprob._lattice_coords((n, n, n), (h, h, h), offset=1.0)
        return pp.ProblemInstance(matrix=A, coords=coords, grid=grid, components=1, rhs=np.zeros(n ** 3),
                                  label="cfg4"), 9, 1e-3, 4
    if cfg == 3:
        n = n or 128
        h = 1.0 / n
        a = 10.0 ** np.random.default_rng(2).uniform(-3, 3, n ** 3)
        fld = pprob.ScalarField(dims=(n, n, n), values=a)
        prob = pprob.darcy_tpfa(fld, spacing=h, dirichlet_face="x-")
        lam = fld.cube()
        ids = np.arange(n ** 3).reshape((n, n, n), order="F")
        extra = np.zeros(n ** 3)
        for axis, side in ((0, -1), (1, 0), (1, -1), (2, 0), (2, -1)):
            s2 = [slice(None)] * 3
            s2[axis] = side
            np.add.at(extra, ids[tuple(s2)].ravel(), 2.0 * lam[tuple(s2)].ravel() * h)
        A = (prob.matrix + sp.diags(extra)).tocsr()
        return pp.ProblemInstance(matrix=A, coords=prob.coords, grid=prob.grid, components=1,
                                  rhs=np.zeros(n ** 3), label="cfg3"), 9, 1e-2, 3
    if cfg == 5:
        ne = n or 64
        h = 1.0 / ne
        vx = ne + 1
        nv = vx ** 3
        E = 10.0 ** np.random.default_rng(5).uniform(-1, 1, ne ** 3)
        nu = 0.3
        lam = E * nu / ((1 + nu) * (1 - 2 * nu))
        mu = E / (2 * (1 + nu))
        K1 = pprob.hex_element_stiffness((h, h, h), 1.0, 0.0)
        K2 = pprob.hex_element_stiffness((h, h, h), 0.0, 1.0)
        e = np.arange(ne ** 3)
        ei, ej, ek = e % ne, (e // ne) % ne, e // (ne * ne)
        corners = np.empty((len(e), 8), dtype=np.int64)
        for c in range(8):
            corners[:, c] = (ei + (c & 1)) + vx * ((ej + ((c >> 1) & 1)) + vx * (ek + ((c >> 2) & 1)))
        dofs = np.concatenate([corners + comp * nv for comp in range(3)], axis=1)
        data = lam[:, None, None] * K1 + mu[:, None, None] * K2
        K = sp.coo_matrix((data.ravel(), (np.repeat(dofs, 24, axis=1).ravel(), np.tile(dofs, (1, 24)).ravel())),
                          shape=(3 * nv, 3 * nv)).tocsr()
        vids = np.arange(nv)
        free_v = vids[vids % vx != 0]
        free = np.concatenate([free_v + c * nv for c in range(3)])
        A = K[free][:, free].tocsr()
        coords = pprob._lattice_coords((vx, vx, vx), (h, h, h), offset=0.0)[free_v]
        grid = pp.CartesianGrid(dims=(vx - 1, vx, vx), spacing=(h, h, h), components_per_vertex=3)
        return pp.ProblemInstance(matrix=A, coords=coords, grid=grid, components=3, rhs=np.zeros(A.shape[0]),
                                  label="cfg5"), 6, 1e-2, 6
    raise ValueError(cfg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=4)
    ap.add_argument("--n", type=int, default=None, help="smaller grid (sample); default: the BASELINE size")
    args = ap.parse_args()
    pp = load_reference()
    import numpy as np

    t = time.perf_counter()
    prob, b, rank_tol, seed = build(pp, args.cfg, args.n)
    t_gen = time.perf_counter() - t
    A = prob.matrix
    rhs = np.random.default_rng(seed).uniform(-1.0, 1.0, prob.n)
    t = time.perf_counter()
    P = pp.factorize(prob, scheme="nest-2-2", degree=1, b=b, rank_tol=rank_tol)
    t_f = time.perf_counter() - t
    t = time.perf_counter()
    x, rep = pp.pcg(lambda v: A @ v, rhs, precond=P.apply_inverse, tol=1e-12)
    t_s = time.perf_counter() - t
    try:
        from threadpoolctl import threadpool_info

        blas = [{k: i.get(k) for k in ("internal_api", "num_threads", "version")} for i in threadpool_info()]
    except Exception:
        blas = None
    print(json.dumps({
        "cfg": args.cfg, "n": int(prob.n), "grid": list(prob.grid.dims), "b": b, "rank_tol": rank_tol,
        "t_generate_s": t_gen, "t_factor_s": t_f, "t_solve_s": t_s, "iterations": int(rep.iterations),
        "converged": bool(rep.converged), "final_rel_residual": float(rep.final_rel_residual),
        "flops_factorize": int(P.stats["flops_factorize"]), "flops_apply": int(P.stats["flops_apply"]),
        "factors": int(P.stats["factors"]), "polyprec": pp.__version__,
        "openblas_num_threads": os.environ.get("OPENBLAS_NUM_THREADS"), "blas": blas,
        "cpu_count": os.cpu_count(), "host": os.uname().nodename,
    }), flush=True)


if __name__ == "__main__":
    main()
