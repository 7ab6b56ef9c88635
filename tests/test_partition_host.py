"""Host-side structure: the product's per-axis hierarchy is bit-identical to
the reference's (golden) and to the oracle's lexsort restatement."""
import numpy as np
import pytest

from conftest import Golden, golden_names
from oracle import sgf_oracle as O
from paper_1907_03406_b200 import partition as Pm
from paper_1907_03406_b200.partition import CartesianGrid


def product_levels(g):
    grid = CartesianGrid(tuple(int(d) for d in g["dims"]), components_per_vertex=int(g["comps"]))
    b = g.stats["b"]
    builder = Pm.build_general_hierarchy if g.opts.get("scheme") == "gen-all-all" else Pm.build_nested_hierarchy
    return builder(grid, b)


@pytest.mark.parametrize("name", [n for n in golden_names() if n != "cfg2"])
def test_hierarchy_matches_reference(name):
    g = Golden(name)
    H = product_levels(g)
    assert len(H.hlevels) == int(g["h_levels"])
    for t, hl in enumerate(H.hlevels):
        assert np.array_equal(hl.cell_of_vertex(), g[f"h{t}_cov"])
        assert np.array_equal(hl.kind_code, g[f"h{t}_kind"])
        assert np.array_equal(hl.interior.astype(np.int8), g[f"h{t}_interior"])
        if f"h{t}_father" in g:
            assert np.array_equal(hl.father, g[f"h{t}_father"])


@pytest.mark.parametrize("dims,b,nested", [((17, 17, 17), 3, True), ((9, 5, 12), 3, True), ((20, 20, 1), 5, True),
                                           ((10, 7, 9), 3, False), ((40, 33, 28), 9, True)])
def test_hierarchy_matches_oracle(dims, b, nested):
    grid = CartesianGrid(dims)
    H = (Pm.build_nested_hierarchy if nested else Pm.build_general_hierarchy)(grid, b)
    ref = O.hierarchy(dims, b, nested)
    assert len(ref) == len(H.hlevels)
    for t, (hl, rl) in enumerate(zip(H.hlevels, ref)):
        assert hl.ncells == len(rl.vertices)
        cov = hl.cell_of_vertex()
        for c, verts in enumerate(rl.vertices):
            assert np.array_equal(np.sort(np.flatnonzero(cov == c)), verts)
            assert np.array_equal(hl.cell_vertices(c), verts)
        assert [Pm.KIND_NAMES.get(int(k), "general") for k in hl.kind_code] == rl.kinds
        if rl.father:
            assert all(int(hl.father[c]) == f for c, f in rl.father.items())


def test_level1_unknowns_component_major():
    grid = CartesianGrid((6, 5, 4), components_per_vertex=3)
    H = Pm.build_nested_hierarchy(grid, 3)
    unk, ptr = Pm.level1_unknowns(H)
    assert np.array_equal(np.sort(unk), np.arange(grid.n_unknowns))
    for c in range(H.hlevels[0].ncells):
        cell = H.levels[0].cells[c]
        assert np.array_equal(unk[ptr[c]:ptr[c + 1]], Pm.expand_to_unknowns(cell, grid))


def test_grid_too_small():
    from paper_1907_03406_b200.errors import GridTooSmallError
    with pytest.raises(GridTooSmallError):
        Pm.build_nested_hierarchy(CartesianGrid((2, 2, 2)), 3)
    with pytest.raises(ValueError):
        Pm.build_nested_hierarchy(CartesianGrid((8, 8, 8)), 1)


def test_large_hierarchy_is_fast():
    import time
    t = time.perf_counter()
    H = Pm.build_nested_hierarchy(CartesianGrid((128, 128, 128)), 9)
    unk, ptr = Pm.level1_unknowns(H)
    assert [h.ncells for h in H.hlevels] == [24389, 3375, 343, 27, 1]
    assert time.perf_counter() - t < 10.0


@pytest.mark.parametrize("degree,comps", [(0, 1), (1, 1), (2, 1), (1, 3), (2, 3)])
def test_basis_bitwise_matches_oracle(degree, comps):
    from paper_1907_03406_b200.basis import build_polynomial_basis
    rng = np.random.default_rng(degree + 7 * comps)
    coords = rng.uniform(-2, 3, (57, 3))
    coords[:, 2] = 0.0 if degree == 1 else coords[:, 2]      # a zero column
    B = build_polynomial_basis(coords, degree, comps)
    assert np.array_equal(B.Pi, O.poly_basis(coords, degree, comps))


def test_level1_unknowns_native_matches_numpy():
    """The native cell expansion (sgf_cell_unknowns) equals the numpy one."""
    from paper_1907_03406_b200.partition import (CartesianGrid, build_general_hierarchy, build_nested_hierarchy,
                                                 level1_unknowns, level1_unknowns_numpy)
    for dims, comps, b, gen in [((33, 17, 9), 1, 3, False), ((30, 17, 9), 3, 3, False), ((40, 40, 1), 1, 9, False),
                                ((20, 20, 20), 1, 4, True), ((13, 11, 7), 3, 6, False)]:
        g = CartesianGrid(dims=dims, components_per_vertex=comps)
        h = (build_general_hierarchy if gen else build_nested_hierarchy)(g, b)
        a, p = level1_unknowns(h)
        a2, p2 = level1_unknowns_numpy(h)
        assert np.array_equal(a, a2) and np.array_equal(p, p2)
