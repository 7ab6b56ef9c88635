"""The CPU oracle is pinned against fixtures produced by the reference itself."""
import numpy as np
import pytest

from conftest import Golden, golden_names
from oracle import sgf_oracle as O

SMALL = [n for n in golden_names(full=False) if n not in ("p3d40_b9",)]


def run_oracle(g, replay=True):
    return O.factorize(g.matrix(), g["coords"], tuple(int(d) for d in g["dims"]), int(g["comps"]),
                       replay_perms=g.perms() if replay else None, **g.opts)


@pytest.mark.parametrize("name", SMALL)
def test_oracle_matches_reference(name):
    g = Golden(name)
    P = run_oracle(g)
    assert P.stats == g.stats                                  # flops, ranks, peak bytes: exact
    assert [tuple(e) for e in P.rank_trace] == g.trace()
    for (lv, nd, r), a, b in zip(g.trace(), P.perms, g.perms()):
        assert np.array_equal(a[:r], b[:r])      # pivots past the rank are not meaningful
    y = P.apply_inverse(g["rhs"])
    ref = g["apply_inverse"]
    assert np.linalg.norm(y - ref) <= 1e-11 * np.linalg.norm(ref)
    w = P.apply_operator(g["rhs"])
    assert np.linalg.norm(w - g["apply_operator"]) <= 1e-11 * np.linalg.norm(g["apply_operator"])
    # apply_half_inverse: its dropped coordinates (idx[r:] of every
    # compression) are Q2^T L^-1 x_B, and the reference's Q2 is fixed by
    # rounding (columns past the numerical rank); every other entry, and the
    # norm of each dropped chunk, is invariant
    h = P.half_inverse(g["rhs"])
    ref = g["half_inverse"]
    keep = np.ones(len(h), bool)
    for f in P.factors:
        if f.kind == "comp":
            d = f.idx[f.retained:]
            keep[d] = False
            assert abs(np.linalg.norm(h[d]) - np.linalg.norm(ref[d])) <= 1e-10 * np.linalg.norm(ref)
    assert np.linalg.norm(h[keep] - ref[keep]) <= 1e-10 * np.linalg.norm(ref[keep])


@pytest.mark.parametrize("name", ["p3d12_b3", "p2d32_b5", "elast3", "p3d9_gen_d1"])
def test_oracle_factor_entries(name):
    g = Golden(name)
    P = run_oracle(g)
    assert len(P.factors) == int(g["nfactors"])
    for k, f in enumerate(P.factors):
        typ = str(g[f"f{k}_type"])
        assert {"elim": "EliminationFactor", "comp": "CompressionFactor", "dense": "DenseFactor"}[f.kind] == typ
        assert np.array_equal(f.idx, g[f"f{k}_idx"])
        L = g[f"f{k}_L"]
        assert np.abs(f.L - L).max() <= 1e-12 * max(np.abs(L).max(), 1.0)
        if typ == "EliminationFactor" and len(g[f"f{k}_Eidx"]):
            E = np.vstack([e for _, e in f.couplings])
            assert np.array_equal(np.concatenate([i for i, _ in f.couplings]), g[f"f{k}_Eidx"])
            assert np.abs(E - g[f"f{k}_E"]).max() <= 1e-12 * max(np.abs(E).max(), 1.0)
        if typ == "CompressionFactor":
            assert f.retained == int(g[f"f{k}_r"])
            r = f.retained
            assert np.abs(f.Q[:, :r] - g[f"f{k}_Q"][:, :r]).max() <= 1e-10


@pytest.mark.parametrize("name", ["p3d12_b3", "cfg1", "aniso14", "tpfa12"])
def test_oracle_pcg_history(name):
    g = Golden(name)
    P = run_oracle(g)
    A = g.matrix()
    x, rep = O.pcg(A, g["rhs"], P.apply_inverse, tol=1e-12)
    assert rep.iterations == int(g["pcg_iters"])
    h = np.array(rep.residual_history)
    ref = g["pcg_hist"]
    assert len(h) == len(ref)
    # all entries but the last (rounding-floor true residual) agree tightly
    assert np.all(np.abs(h[:-1] - ref[:-1]) <= 1e-10 * np.maximum(ref[:-1], 1e-300) + 1e-14)


def test_free_running_oracle_iterations():
    # without pivot replay the oracle may resolve rounding-level pivot ties
    # differently; ranks and iteration counts still agree
    g = Golden("cfg1")
    P = run_oracle(g, replay=False)
    assert [tuple(e) for e in P.rank_trace] == g.trace()
    x, rep = O.pcg(g.matrix(), g["rhs"], P.apply_inverse, tol=1e-12)
    assert abs(rep.iterations - int(g["pcg_iters"])) <= 1


def test_oracle_errors():
    import scipy.sparse as sp
    A = sp.csr_matrix(-np.eye(4))
    with pytest.raises(O.OracleNotSPD):
        O.chol_lower(-np.eye(4), O.Tally())
    with pytest.raises(ValueError):
        O.Blocks.from_csr(sp.csr_matrix(np.array([[1.0, 2.0], [0.0, 1.0]])), {0: np.arange(2)})
    with pytest.raises(O.OracleIndefinite):
        O.pcg(A, np.ones(4), None, tol=1e-10)


def test_qrcp_known_answers():
    t = O.Tally()
    assert O.qrcp(np.eye(3), 1e-10, t).rank == 3
    assert O.qrcp(np.array([[1.0, 2.0], [2.0, 4.0]]), 1e-10, t).rank == 1
    D = np.diag([1.0, 1e-3, 1e-12])
    assert O.qrcp(D, 1e-10, t).rank == 2
    assert O.qrcp(D, 1e-14, t).rank == 3
    A = np.random.default_rng(3).standard_normal((9, 5))
    q = O.qrcp(A, 1e-10, t)
    assert np.abs(q.Q.T @ q.Q - np.eye(9)).max() <= 1e-12
    assert np.abs(A[:, q.perm] - q.Q[:, :5] @ q.R).max() <= 1e-12 * np.abs(A).max()
