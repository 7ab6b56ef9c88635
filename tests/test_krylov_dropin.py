"""`pcg` as a drop-in: the reference's TestPCG cases (reference
tests/test_krylov.py:11-87) and the bench call pattern
`pcg(lambda v: A @ v, rhs, precond=P.apply_inverse, tol=1e-12)` (reference
bench.py:163-164), run against the product on the GPU, plus the operator
classification (krylov.py:28-31 `_as_linop`) and stream ordering with torch."""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

sgf = pytest.importorskip("paper_1907_03406_b200")
from paper_1907_03406_b200 import krylov as K  # noqa: E402
from paper_1907_03406_b200.errors import IndefiniteDetectedError  # noqa: E402

pcg, factorize, poisson7 = sgf.pcg, sgf.factorize, sgf.poisson7


class TestPCG:
    def test_identity_one_iteration(self):
        b = np.arange(1.0, 6.0)
        x, rep = pcg(np.eye(5), b)
        assert rep.iterations == 1
        assert rep.converged
        assert np.allclose(x, b)

    def test_zero_rhs(self):
        x, rep = pcg(np.eye(4), np.zeros(4))
        assert rep.iterations == 0
        assert rep.residual_history == [0.0]
        assert rep.converged
        assert np.allclose(x, 0.0)

    def test_exact_preconditioner_two_iterations(self):
        prob = poisson7(11)
        P = factorize(prob, scheme="nest-2-2", compression=False)
        rng = np.random.default_rng(0)
        b = rng.uniform(-1, 1, prob.n)
        x, rep = pcg(lambda v: prob.matrix @ v, b, precond=P.apply_inverse, tol=1e-10)
        assert rep.converged
        assert rep.iterations <= 2

    def test_history_shape_and_first_entry(self):
        prob = poisson7(6)
        rng = np.random.default_rng(1)
        b = rng.standard_normal(prob.n)
        x, rep = pcg(lambda v: prob.matrix @ v, b, tol=1e-8)
        assert rep.residual_history[0] == 1.0
        assert len(rep.residual_history) == rep.iterations + 1
        assert rep.converged
        assert rep.final_rel_residual <= 1e-8

    def test_final_residual_matches_recomputation(self):
        prob = poisson7(8)
        rng = np.random.default_rng(2)
        b = rng.standard_normal(prob.n)
        x, rep = pcg(lambda v: prob.matrix @ v, b, tol=1e-9)
        check = np.linalg.norm(b - prob.matrix @ x) / np.linalg.norm(b)
        assert abs(rep.final_rel_residual - check) <= 1e-12

    def test_unpreconditioned_matches_direct(self):
        prob = poisson7(6)
        rng = np.random.default_rng(3)
        b = rng.standard_normal(prob.n)
        x, rep = pcg(lambda v: prob.matrix @ v, b, tol=1e-12)
        want = np.linalg.solve(prob.matrix.toarray(), b)
        assert np.linalg.norm(x - want) <= 1e-9 * np.linalg.norm(want)

    def test_indefinite_operator_detected(self):
        A = np.diag([1.0, -1.0])
        with pytest.raises(IndefiniteDetectedError):
            pcg(A, np.array([1.0, 1.0]))

    def test_indefinite_preconditioner_detected(self):
        A = np.eye(3) * 2.0
        M = np.diag([1.0, 1.0, -1.0])
        with pytest.raises(IndefiniteDetectedError):
            pcg(A, np.array([0.1, 0.1, 1.0]), precond=M)

    def test_maxit_reported_unconverged(self):
        prob = poisson7(8)
        rng = np.random.default_rng(4)
        b = rng.standard_normal(prob.n)
        x, rep = pcg(lambda v: prob.matrix @ v, b, tol=1e-14, maxit=3)
        assert not rep.converged
        assert rep.iterations == 3

    def test_true_residual_recompute_guards_drift(self):
        prob = poisson7(10)
        rng = np.random.default_rng(5)
        b = rng.standard_normal(prob.n)
        x, rep = pcg(lambda v: prob.matrix @ v, b, tol=1e-10, true_residual_every=10)
        assert rep.converged
        assert np.linalg.norm(b - prob.matrix @ x) / np.linalg.norm(b) <= 1e-10

    def test_report_serializable(self):
        import dataclasses
        import json

        prob = poisson7(4)
        _, rep = pcg(lambda v: prob.matrix @ v, np.ones(prob.n), tol=1e-8)
        text = json.dumps(dataclasses.asdict(rep))
        assert json.loads(text)["iterations"] == rep.iterations


def _reference_pcg(A, b, M, tol=1e-10, maxit=5000, true_every=50):
    """The reference recurrence (krylov.py:34-102) in numpy, for comparing
    the opaque-callback path."""
    bnorm = np.linalg.norm(b)
    x = np.zeros_like(b)
    r = b.copy()
    hist = [1.0]
    z = M(r)
    rz = r @ z
    p = z.copy()
    it = 0
    while it < maxit:
        it += 1
        Ap = A(p)
        alpha = rz / (p @ Ap)
        x += alpha * p
        r -= alpha * Ap
        if it % true_every == 0:
            r = b - A(x)
        rel = np.linalg.norm(r) / bnorm
        if rel <= tol:
            r = b - A(x)
            rel = np.linalg.norm(r) / bnorm
            hist.append(rel)
            if rel <= tol:
                break
        else:
            hist.append(rel)
        z = M(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, hist, it


def test_operator_classification():
    """Which path each operator form takes (none of them silently on the CPU
    except opaque user callables, whose own code runs where the user wrote it)."""
    prob = poisson7(6)
    A = prob.matrix
    P = factorize(prob)
    assert K._classify(A, "m").kind == "csr"
    assert K._classify(A.toarray(), "m").kind == "csr"
    assert K._classify(lambda v: A @ v, "m").kind == "csr"
    assert K._classify(lambda v: A.dot(v), "m").kind == "csr"
    assert K._classify(P, "p").kind == "precond"
    assert K._classify(P.apply_inverse, "p").kind == "precond"
    assert K._classify(lambda v: P.apply_inverse(v), "p").kind == "precond"
    assert K._classify(lambda v: P @ v, "p").kind == "precond"
    op = K._classify(P.apply_operator, "m")
    assert op.kind == "precond" and op.apply_op == 3
    assert K._classify(lambda v: 2.0 * (A @ v), "m").kind == "host"
    assert K._classify(sp.linalg.aslinearoperator(A), "m").kind == "host"


def test_bench_call_pattern_equals_device_path():
    """reference bench.py:163-164 call pattern == the CSR + Preconditioner
    call (the probe routes the lambda to the same device path: bitwise)."""
    prob = poisson7(12)
    P = factorize(prob, b=3, rank_tol=1e-2)
    rhs = np.random.default_rng(1).uniform(-1, 1, prob.n)
    A = prob.matrix
    x1, r1 = pcg(lambda v: A @ v, rhs, precond=P.apply_inverse, tol=1e-12)
    x2, r2 = pcg(A, rhs, precond=P, tol=1e-12)
    assert r1.residual_history == r2.residual_history
    assert np.array_equal(x1, x2)


def test_opaque_callbacks_follow_the_reference_recurrence():
    """A callable the probe cannot see into (a scaled operator, a Jacobi
    preconditioner closure) runs on host copies each iteration; the history
    follows the reference recurrence."""
    prob = poisson7(9)
    A = prob.matrix
    d = A.diagonal()
    rhs = np.random.default_rng(2).uniform(-1, 1, prob.n)
    Aop = lambda v: 2.0 * (A @ v)  # noqa: E731
    Mop = lambda v: v / d  # noqa: E731
    x, rep = pcg(Aop, rhs, precond=Mop, tol=1e-10, true_residual_every=7)
    xr, hr, itr = _reference_pcg(Aop, rhs, Mop, tol=1e-10, true_every=7)
    assert rep.iterations == itr
    h = np.array(rep.residual_history)
    assert np.all(np.abs(h[:-1] - np.array(hr)[:-1]) <= 1e-9 * np.array(hr)[:-1] + 1e-15)
    assert np.linalg.norm(x - xr) <= 1e-9 * np.linalg.norm(xr)
    # a preconditioner given as another Preconditioner method runs on the device
    P = factorize(prob)
    x, rep = pcg(A, rhs, precond=P.apply_operator, tol=1e-8, maxit=2000)
    assert rep.converged


def test_callback_errors_propagate():
    prob = poisson7(5)

    def bad(v):
        raise KeyError("user operator failed")

    with pytest.raises(KeyError):
        pcg(bad, np.ones(prob.n))
    with pytest.raises(sgf.ShapeMismatchError):
        pcg(lambda v: np.ones(3), np.ones(prob.n))  # wrong output length


def test_device_tensor_inputs_are_stream_ordered():
    """A right-hand side still being produced by a torch kernel on torch's
    stream is read only after that kernel finished (the native
    stream is non-blocking)."""
    import torch

    prob = poisson7(20)
    P = factorize(prob, rank_tol=1e-2)
    A = sgf.DeviceCSR(prob.matrix)
    rhs = np.random.default_rng(3).uniform(-1, 1, prob.n)
    want = P.apply_inverse(rhs)
    big = torch.randn(4096, 4096, device="cuda", dtype=torch.float64)
    for _ in range(3):
        torch.cuda.synchronize()
        # a long torch kernel, then the input written behind it on torch's stream
        big @ big
        x = torch.tensor(rhs, device="cuda") * 1.0
        y = P.apply_inverse(x)
        assert np.linalg.norm(y.cpu().numpy() - want) <= 1e-14 * np.linalg.norm(want)
        big @ big
        b = torch.tensor(rhs, device="cuda") * 1.0
        xs, rep = pcg(A, b, precond=P, tol=1e-10)
        assert rep.converged


def test_rank_trace_outside_lowrank_is_rejected():
    """reference factorization.py:543-549: trace entries that are never
    replayed (polynomial / exact mode) raise RuntimeError."""
    prob = poisson7(12)
    P = factorize(prob, b=3, rank_tol=1e-2)
    assert len(P.rank_trace) > 0
    with pytest.raises(RuntimeError, match="unreplayed"):
        factorize(prob, b=3, rank_tol=1e-2, rank_trace=P.rank_trace)
    factorize(prob, b=3, rank_tol=1e-2, rank_trace=sgf.RankTrace())  # empty: fine


def test_forced_rank_clipping_warns():
    """reference factorization.py:334-336: warnings.warn when a replayed rank
    exceeds the node size."""
    prob = poisson7(9)
    P = factorize(prob, scheme="gen-all-all", degree=0)
    big = sgf.RankTrace([(lv, nd, 10 ** 6) for lv, nd, r in P.rank_trace.entries])
    with pytest.warns(UserWarning, match="clipping"):
        factorize(prob, scheme="gen-all-all", degree=0, mode="lowrank", rank_trace=big)
