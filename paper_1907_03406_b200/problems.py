"""Problem instances and the synthetic generators of the BASELINE configs.

`ProblemInstance` mirrors the reference container (`problems.py:26-58`):
CSR matrix, per-vertex coordinates, CartesianGrid, components, rhs, label.
The generators are harness code (the reference's `problems.py` is out of the
hot-path scope); they build the five BASELINE
configs exactly as SURVEY.md section 8(d) specifies them:

  cfg1 poisson2d(128)                    2-D 5-point, h = 1/129
  cfg2 poisson7(64, spacing=1/65)        3-D 7-point
  cfg3 tpfa_dirichlet(128, seed=2)       cell-centred TPFA, a = 10^U[-3,3], Dirichlet on 6 faces
  cfg4 anisotropic7(128, 1e-3)           Tx + Ty + 1e-3 Tz
  cfg5 elasticity_cube(64, seed=5)       Q1 hexahedra, E = 10^U[-1,1], nu = 0.3, x = 0 clamped
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .errors import DimensionMismatchError, NotSymmetricError
from .partition import CartesianGrid


@dataclass
class ProblemInstance:
    matrix: sp.csr_matrix
    coords: np.ndarray
    grid: CartesianGrid
    components: int
    rhs: np.ndarray
    label: str
    check_symmetry: bool = True

    def __post_init__(self):
        n = self.grid.n_unknowns
        if self.matrix.shape != (n, n):
            raise DimensionMismatchError(f"matrix is {self.matrix.shape}, grid implies {n} unknowns")
        if self.coords.shape != (self.grid.n_vertices, 3):
            raise DimensionMismatchError(
                f"coords are {self.coords.shape}, expected ({self.grid.n_vertices}, 3)")
        if self.check_symmetry:
            asym = abs(self.matrix - self.matrix.T)
            if asym.nnz and asym.max() > 1e-12 * abs(self.matrix).max():
                raise NotSymmetricError(f"matrix asymmetry {asym.max():.2e}")

    @property
    def n(self):
        return self.matrix.shape[0]


def _lattice(dims, spacing, offset):
    """Vertex coordinates, x fastest: id = i + nx*(j + ny*k)."""
    nx, ny, nz = dims
    hx, hy, hz = spacing
    c = np.empty((nx * ny * nz, 3))
    c[:, 0] = np.tile((np.arange(nx) + offset) * hx, ny * nz)
    c[:, 1] = np.repeat(np.tile((np.arange(ny) + offset) * hy, nz), nx)
    c[:, 2] = np.repeat((np.arange(nz) + offset) * hz, nx * ny)
    return c


def _lap1d(n, h):
    return sp.diags([np.full(n - 1, -1.0 / h ** 2), np.full(n, 2.0 / h ** 2),
                     np.full(n - 1, -1.0 / h ** 2)], [-1, 0, 1], format="csr")


def _kron3(Tx, Ty, Tz, nx, ny, nz):
    Ix, Iy, Iz = (sp.identity(m, format="csr") for m in (nx, ny, nz))
    return (sp.kron(Iz, sp.kron(Iy, Tx)) + sp.kron(Iz, sp.kron(Ty, Ix))
            + sp.kron(Tz, sp.kron(Iy, Ix))).tocsr()


def poisson7(nx, ny=None, nz=None, spacing=1.0):
    """3-D 7-point Poisson with folded Dirichlet boundary (reference
    problems.py:90-117 conventions: coords offset 1, x fastest)."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    if min(nx, ny, nz) < 2:
        raise ValueError("each axis needs at least 2 interior vertices")
    h = (float(spacing),) * 3 if np.isscalar(spacing) else tuple(float(s) for s in spacing)
    A = _kron3(_lap1d(nx, h[0]), _lap1d(ny, h[1]), _lap1d(nz, h[2]), nx, ny, nz)
    grid = CartesianGrid(dims=(nx, ny, nz), spacing=h)
    return ProblemInstance(A, _lattice((nx, ny, nz), h, 1.0), grid, 1,
                           np.ones(grid.n_unknowns), f"poisson-{nx}x{ny}x{nz}")


def poisson2d(n, spacing=None):
    """cfg1: 2-D 5-point Laplacian on an n x n interior grid (nz = 1)."""
    h = 1.0 / (n + 1) if spacing is None else float(spacing)
    T = _lap1d(n, h)
    I = sp.identity(n, format="csr")
    A = (sp.kron(I, T) + sp.kron(T, I)).tocsr()
    grid = CartesianGrid(dims=(n, n, 1), spacing=(h, h, h))
    return ProblemInstance(A, _lattice((n, n, 1), (h, h, h), 1.0), grid, 1,
                           np.ones(n * n), f"poisson2d-{n}")


def anisotropic7(n, eps_z=1e-3):
    """cfg4: diag(1, 1, eps_z) diffusion, 7-point, h = 1/(n+1)."""
    h = 1.0 / (n + 1)
    A = _kron3(_lap1d(n, h), _lap1d(n, h), eps_z * _lap1d(n, h), n, n, n)
    grid = CartesianGrid(dims=(n, n, n), spacing=(h, h, h))
    return ProblemInstance(A, _lattice((n, n, n), (h, h, h), 1.0), grid, 1,
                           np.ones(n ** 3), f"aniso-{n}-{eps_z:g}")


def tpfa_dirichlet(n, seed=2, log_range=3.0):
    """cfg3: cell-centred two-point flux on n^3 cells of the unit cube, cell
    coefficient a = 10^U[-log_range, log_range] (x-fastest cell order),
    harmonic-mean face transmissibilities, Dirichlet on all six faces by the
    half-cell term 2*a*geo (reference darcy_tpfa conventions,
    problems.py:234-299, with the x- face term added first and the other
    five after it in the order x+, y-, y+, z-, z+)."""
    h = 1.0 / n
    a = 10.0 ** np.random.default_rng(seed).uniform(-log_range, log_range, n ** 3)
    lam = a.reshape((n, n, n), order="F")
    ids = np.arange(n ** 3).reshape((n, n, n), order="F")
    N = n ** 3
    diag = np.zeros(N)
    rows, cols, vals = [], [], []
    geo = h * h / h
    for axis in range(3):
        sa = [slice(None)] * 3
        sb = [slice(None)] * 3
        sa[axis] = slice(None, -1)
        sb[axis] = slice(1, None)
        la, lb = lam[tuple(sa)].ravel(), lam[tuple(sb)].ravel()
        ia, ib = ids[tuple(sa)].ravel(), ids[tuple(sb)].ravel()
        T = 2.0 * la * lb / (la + lb) * geo
        rows.append(ia)
        cols.append(ib)
        vals.append(-T)
        np.add.at(diag, ia, T)
        np.add.at(diag, ib, T)
    sl = [slice(None)] * 3
    sl[0] = 0
    np.add.at(diag, ids[tuple(sl)].ravel(), 2.0 * lam[tuple(sl)].ravel() * geo)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals)
    A = sp.coo_matrix((np.concatenate([vals, vals, diag]),
                       (np.concatenate([rows, cols, np.arange(N)]),
                        np.concatenate([cols, rows, np.arange(N)]))), shape=(N, N)).tocsr()
    extra = np.zeros(N)
    for axis, side in ((0, -1), (1, 0), (1, -1), (2, 0), (2, -1)):
        s2 = [slice(None)] * 3
        s2[axis] = side
        np.add.at(extra, ids[tuple(s2)].ravel(), 2.0 * lam[tuple(s2)].ravel() * geo)
    A = (A + sp.diags(extra)).tocsr()
    grid = CartesianGrid(dims=(n, n, n), spacing=(h, h, h))
    return ProblemInstance(A, _lattice((n, n, n), (h, h, h), 0.5), grid, 1,
                           np.zeros(N), f"tpfa-{n}-s{seed}")


_GP = 1.0 / math.sqrt(3.0)
_CORNER = np.array([[(c >> s) & 1 for s in (0, 1, 2)] for c in range(8)], dtype=float) * 2.0 - 1.0


def hex_stiffness(h, lam, mu):
    """24x24 trilinear hexahedron stiffness, component-grouped dofs, 2x2x2
    Gauss (restates reference problems.py:311-351)."""
    hx, hy, hz = (h, h, h) if np.isscalar(h) else h
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[np.arange(3), np.arange(3)] += 2.0 * mu
    D[np.arange(3, 6), np.arange(3, 6)] = mu
    K = np.zeros((24, 24))
    w = hx * hy * hz / 8.0
    for gz in (-_GP, _GP):
        for gy in (-_GP, _GP):
            for gx in (-_GP, _GP):
                s = _CORNER
                dN = np.empty((8, 3))
                dN[:, 0] = 0.125 * s[:, 0] * (1 + s[:, 1] * gy) * (1 + s[:, 2] * gz) * (2.0 / hx)
                dN[:, 1] = 0.125 * s[:, 1] * (1 + s[:, 0] * gx) * (1 + s[:, 2] * gz) * (2.0 / hy)
                dN[:, 2] = 0.125 * s[:, 2] * (1 + s[:, 0] * gx) * (1 + s[:, 1] * gy) * (2.0 / hz)
                B = np.zeros((6, 24))
                B[0, 0:8] = dN[:, 0]
                B[1, 8:16] = dN[:, 1]
                B[2, 16:24] = dN[:, 2]
                B[3, 0:8], B[3, 8:16] = dN[:, 1], dN[:, 0]
                B[4, 8:16], B[4, 16:24] = dN[:, 2], dN[:, 1]
                B[5, 0:8], B[5, 16:24] = dN[:, 2], dN[:, 0]
                K += w * (B.T @ D @ B)
    return 0.5 * (K + K.T)


def elasticity_cube(ne, seed=5, nu=0.3, log_range=1.0):
    """cfg5: Q1 elasticity on ne^3 elements of the unit cube, per-element
    Young's modulus 10^U[-log_range, log_range] (element order i fastest),
    face x = 0 clamped by removing its rows/columns, dofs component-major."""
    h = 1.0 / ne
    vx = vy = vz = ne + 1
    nv = vx * vy * vz
    E = 10.0 ** np.random.default_rng(seed).uniform(-log_range, log_range, ne ** 3)
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    K1 = hex_stiffness(h, 1.0, 0.0)
    K2 = hex_stiffness(h, 0.0, 1.0)
    e = np.arange(ne ** 3)
    ei, ej, ek = e % ne, (e // ne) % ne, e // (ne * ne)
    corners = np.empty((len(e), 8), dtype=np.int64)
    for c in range(8):
        corners[:, c] = (ei + (c & 1)) + vx * ((ej + ((c >> 1) & 1)) + vy * (ek + ((c >> 2) & 1)))
    dofs = np.concatenate([corners + k * nv for k in range(3)], axis=1)
    data = lam[:, None, None] * K1 + mu[:, None, None] * K2
    K = sp.coo_matrix((data.ravel(), (np.repeat(dofs, 24, axis=1).ravel(),
                                      np.tile(dofs, (1, 24)).ravel())),
                      shape=(3 * nv, 3 * nv)).tocsr()
    vids = np.arange(nv)
    free_v = vids[vids % vx != 0]
    free = np.concatenate([free_v + k * nv for k in range(3)])
    A = K[free][:, free].tocsr()
    coords = _lattice((vx, vy, vz), (h, h, h), 0.0)[free_v]
    grid = CartesianGrid(dims=(vx - 1, vy, vz), spacing=(h, h, h), components_per_vertex=3)
    return ProblemInstance(A, coords, grid, 3, np.zeros(A.shape[0]), f"elast-{ne}-s{seed}")


# BASELINE.json configs: generator, b, rank_tol, rhs seed
CONFIGS = {
    1: dict(make=lambda: poisson2d(128), b=9, rank_tol=1e-2, seed=0, name="cfg1-poisson2d-128"),
    2: dict(make=lambda: poisson7(64, spacing=1.0 / 65), b=9, rank_tol=1e-2, seed=1,
            name="cfg2-poisson3d-64"),
    3: dict(make=lambda: tpfa_dirichlet(128, seed=2), b=9, rank_tol=1e-2, seed=3,
            name="cfg3-tpfa-hc-128"),
    4: dict(make=lambda: anisotropic7(128, 1e-3), b=9, rank_tol=1e-3, seed=4,
            name="cfg4-aniso-128"),
    5: dict(make=lambda: elasticity_cube(64, seed=5), b=6, rank_tol=1e-2, seed=6,
            name="cfg5-elasticity-64"),
}


def config_rhs(n, seed):
    """RHS i.i.d. uniform[-1, 1] (reference bench.py:161-162)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)
