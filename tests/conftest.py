import json
import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsgf.so")


@pytest.fixture(autouse=True)
def _release_failed_test_frames(request):
    """pytest keeps a failed test's traceback in sys.last_traceback (for
    post-mortem debugging); its frames hold the test's locals, e.g. a
    full-size Preconditioner with tens of GB of factors in HBM, which would
    make every later full-size test fail with out-of-memory.  Drop it after
    each test."""
    yield
    import gc

    for k in ("last_type", "last_value", "last_traceback", "last_exc"):
        if hasattr(sys, k):
            setattr(sys, k, None)
    if request.node.get_closest_marker("gpu") is not None:
        gc.collect()


class Golden:
    """One reference-generated fixture (tests/golden/make_golden.py)."""

    def __init__(self, name):
        self.name = name
        self.z = np.load(os.path.join(GOLDEN, name + ".npz"))
        self.opts = json.loads(str(self.z["opts"]))
        self.stats = json.loads(str(self.z["stats"]))

    def __getitem__(self, k):
        return self.z[k]

    def __contains__(self, k):
        return k in self.z.files

    @property
    def n(self):
        return len(self.z["rhs"])

    def matrix(self):
        z = self.z
        return sp.csr_matrix((z["data"], z["indices"], z["indptr"]), shape=(self.n, self.n))

    def problem(self):
        from paper_1907_03406_b200.partition import CartesianGrid
        from paper_1907_03406_b200.problems import ProblemInstance

        z = self.z
        grid = CartesianGrid(dims=tuple(int(d) for d in z["dims"]),
                             spacing=tuple(float(s) for s in z["spacing"]),
                             components_per_vertex=int(z["comps"]))
        return ProblemInstance(self.matrix(), z["coords"], grid, int(z["comps"]), z["rhs"], self.name,
                               check_symmetry=False)

    def perms(self):
        z = self.z
        p = z["perm_ptr"]
        return [z["perm_all"][p[i]:p[i + 1]] for i in range(len(p) - 1)]

    def trace(self):
        return [tuple(int(v) for v in e) for e in self.z["rank_trace"]]


def golden_names(full=True):
    """Regular fixtures (the slim full-size ones, FullGolden, are separate)."""
    names = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f[:-4] not in FULL_GOLDEN_MAKERS)
    if not full:
        names = [n for n in names if "data" in np.load(os.path.join(GOLDEN, n + ".npz")).files]
    return names


@pytest.fixture(scope="session")
def goldens():
    return {n: Golden(n) for n in golden_names()}


def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


FULL_GOLDEN_MAKERS = {
    # fixture name -> (product generator, rhs seed); the fixture's matrix
    # digest pins that the generator reproduces the reference's matrix bitwise
    "cfg3_full": ("tpfa_dirichlet", (128,), {"seed": 2}),
    "cfg4_full": ("anisotropic7", (128, 1e-3), {}),
    "cfg5_full": ("elasticity_cube", (64,), {"seed": 5}),
    "tpfa40_b9": ("tpfa_dirichlet", (40,), {"seed": 2}),
}


class FullGolden(Golden):
    """A slim reference fixture at full size (make_golden.py run_full):
    digests, trace, QR permutations, stats, sampled/projected vectors and
    sampled factors; the matrix comes from the product's generator."""

    def problem(self):
        from paper_1907_03406_b200 import problems as Pm

        fn, args, kw = FULL_GOLDEN_MAKERS[self.name]
        return getattr(Pm, fn)(*args, **kw)

    @property
    def n(self):
        return int(self.z["n"])

    def rhs(self):
        return np.random.default_rng(int(self.z["rhs_seed"])).uniform(-1.0, 1.0, self.n)

    def proj(self):
        return np.random.default_rng(7).standard_normal((4, self.n))

    def vec_errors(self, key, y, proj=None):
        """(strided-sample rel error, projection rel error, norm rel error)."""
        z = self.z
        s = z[f"{key}_s"]
        es = np.linalg.norm(y[::32] - s) / np.linalg.norm(s)
        p = (self.proj() if proj is None else proj) @ y
        ep = np.max(np.abs(p - z[f"{key}_p"]) / (np.linalg.norm(z[f"{key}_p"]) + 1e-300))
        en = abs(np.linalg.norm(y) - float(z[f"{key}_norm"])) / float(z[f"{key}_norm"])
        return es, ep, en


def full_golden_names():
    return sorted(n for n in FULL_GOLDEN_MAKERS if os.path.exists(os.path.join(GOLDEN, n + ".npz")))


def hierarchy_digests(problem, scheme, b):
    """sha256 per level of (cell_of_vertex, kind, interior, father) exactly as
    make_golden.hierarchy_digest forms it from the reference hierarchy."""
    from paper_1907_03406_b200 import partition as Pm

    builder = Pm.build_general_hierarchy if scheme == "gen-all-all" else Pm.build_nested_hierarchy
    H = builder(problem.grid, b)
    out = []
    for t, hl in enumerate(H.hlevels):
        parts = [hl.cell_of_vertex().astype(np.int32), hl.kind_code.astype(np.int8), hl.interior.astype(np.int8)]
        if t + 1 < len(H.hlevels):
            parts.append(np.asarray(hl.father).astype(np.int32))
        out.append(array_digest(*parts))
    return out


def array_digest(*arrays):
    import hashlib

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
    return array_digest(A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data.astype(np.float64))
