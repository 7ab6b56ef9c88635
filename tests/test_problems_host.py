"""Config generators reproduce the matrices the golden script built with the
reference's own generator pieces."""
import numpy as np
import pytest

from conftest import Golden
from paper_1907_03406_b200 import problems as pr


def same(A, g, tol=0.0):
    B = g.matrix()
    assert A.shape == B.shape
    D = (A - B).tocoo()
    if tol == 0.0:
        assert D.nnz == 0 or np.abs(D.data).max() == 0.0
    else:
        assert np.abs(D.data).max(initial=0.0) <= tol * abs(B).max()


def test_poisson3d():
    g = Golden("p3d12_b3")
    p = pr.poisson7(12)
    same(p.matrix, g)
    assert np.array_equal(p.coords, g["coords"])


def test_poisson2d():
    g = Golden("p2d32_b5")
    p = pr.poisson2d(32)
    same(p.matrix, g)
    assert np.array_equal(p.coords, g["coords"])
    assert p.grid.dims == (32, 32, 1)


def test_anisotropic():
    g = Golden("aniso14")
    p = pr.anisotropic7(14, 1e-3)
    same(p.matrix, g, 1e-15)
    assert np.array_equal(p.coords, g["coords"])


def test_tpfa_all_dirichlet():
    g = Golden("tpfa12")
    p = pr.tpfa_dirichlet(12, seed=2)
    same(p.matrix, g)
    assert np.array_equal(p.coords, g["coords"])


@pytest.mark.parametrize("ne,name", [(3, "elast3"), (8, "elast8")])
def test_elasticity(ne, name):
    g = Golden(name)
    p = pr.elasticity_cube(ne, seed=5)
    same(p.matrix, g, 1e-14)
    assert np.allclose(p.coords, g["coords"], rtol=0, atol=0)
    assert p.grid.components_per_vertex == 3


def test_config_sizes():
    # sizes quoted by BASELINE.md for the five configs (cheap ones built here)
    p = pr.CONFIGS[1]["make"]()
    assert p.n == 16384 and p.matrix.nnz == 81408
    assert pr.elasticity_cube(4).n == 3 * 4 * 5 * 5
