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
    names = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))
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
