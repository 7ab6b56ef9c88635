"""Cartesian partition hierarchies, computed per axis.

Same cells, ids, kinds, roles and father maps as the reference
(`partition.py:105-242`), but built without a global sort: a cell of the
nested (or general) family is a box whose per-axis extent is one axis
*label* (sep, group).  Because every combination of per-axis labels occurs,
the reference's cell id -- the rank of the vertex label tuple
(sep_x, grp_x, sep_y, grp_y, sep_z, grp_z) in lexicographic order
(`partition.py:142-176`, `np.lexsort(key.T[::-1])` at :154) -- factorises as

    id = rank_x * (T_y * T_z) + rank_y * T_z + rank_z

where rank_a is the rank of the axis label among the T_a distinct labels of
axis a.  Everything below is O(n) integer work; it is checked bit-exactly
against the oracle and the reference's golden hierarchies in tests/.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from .errors import GridTooSmallError

KIND_NAMES = {0: "cell0", 1: "cell1", 2: "cell2", 3: "cell3"}
# integer kind codes shared with the C ABI (include/sgf.h: SGF_KIND_*)
KIND_CODE = {"cell0": 0, "cell1": 1, "cell2": 2, "cell3": 3, "general": 4}


@dataclass(frozen=True)
class CartesianGrid:
    """Vertex lattice with per-axis spacing and unknowns per vertex
    (reference `partition.py:25-46`)."""

    dims: tuple
    spacing: tuple = (1.0, 1.0, 1.0)
    components_per_vertex: int = 1

    def __post_init__(self):
        if len(self.dims) != 3 or any(d < 1 for d in self.dims):
            raise ValueError(f"bad grid dims {self.dims}")
        if len(self.spacing) != 3 or any(h <= 0 for h in self.spacing):
            raise ValueError(f"bad grid spacing {self.spacing}")

    @property
    def n_vertices(self):
        nx, ny, nz = self.dims
        return nx * ny * nz

    @property
    def n_unknowns(self):
        return self.n_vertices * self.components_per_vertex


@dataclass
class Cell:
    """One partition cell (reference `partition.py:49-61`)."""

    id: int
    vertex_ids: np.ndarray
    kind: str
    role: str
    box: tuple

    @property
    def size(self):
        return len(self.vertex_ids)


@dataclass
class Level:
    cells: list
    father: dict = field(default_factory=dict)
    adjacency: set = field(default_factory=set)


class AxisLabels:
    """Distinct labels of one axis at one level, in lexicographic order.

    lo/hi: inclusive index extent of each label; sep: 1 for separator
    layers; rank: label rank of every grid index on this axis."""

    def __init__(self, n, d, nested):
        i = np.arange(n)
        if nested:
            # partition.py:105-111
            sep = ((i + 1) % d == 0).astype(np.int64)
            grp = np.where(sep == 1, (i + 1) // d - 1, i // d)
        else:
            sep = np.zeros(n, dtype=np.int64)          # partition.py:122-124
            grp = i // d
        key = sep * (n + 1) + grp                      # (sep, grp) lexicographic
        uniq, self.rank = np.unique(key, return_inverse=True)
        self.rank = self.rank.astype(np.int64)
        self.sep = (uniq // (n + 1)).astype(np.int64)
        self.grp = (uniq % (n + 1)).astype(np.int64)
        self.count = len(uniq)
        self.lo = np.full(self.count, n, dtype=np.int64)
        self.hi = np.full(self.count, -1, dtype=np.int64)
        np.minimum.at(self.lo, self.rank, i)
        np.maximum.at(self.hi, self.rank, i)
        self.n = n
        self.nested = nested

    def up(self, nxt):
        """Rank at the next level of each label's father label
        (partition.py:114-119 nested, :126-127 general)."""
        s, g = self.sep, self.grp
        if self.nested:
            odd = (g % 2) == 1
            fs = np.where((s == 1) & odd, 1, 0)
            fg = np.where((s == 1) & odd, (g - 1) // 2, g // 2)
        else:
            fs = np.zeros_like(s)
            fg = g // 2
        nk = nxt.sep * (nxt.n + 1) + nxt.grp
        fk = fs * (nxt.n + 1) + fg
        pos = np.searchsorted(nk, fk)
        assert np.all(nk[pos] == fk), "father label missing at next level"
        return pos.astype(np.int64)


class HLevel:
    """One level as arrays: axis label tables, per-cell kind/role codes."""

    def __init__(self, grid, d, nested):
        self.d = d
        self.axes = [AxisLabels(n, d, nested) for n in grid.dims]
        tx, ty, tz = (a.count for a in self.axes)
        self.shape = (tx, ty, tz)
        self.ncells = tx * ty * tz
        cx, cy, cz = np.meshgrid(np.arange(tx), np.arange(ty), np.arange(tz), indexing="ij")
        self.cx, self.cy, self.cz = cx.ravel(), cy.ravel(), cz.ravel()
        ax, ay, az = self.axes
        if nested:
            nsep = ax.sep[self.cx] + ay.sep[self.cy] + az.sep[self.cz]
            self.kind_code = (3 - nsep).astype(np.int32)          # partition.py:131-135
            self.interior = (nsep == 0)
        else:
            self.kind_code = np.full(self.ncells, 4, dtype=np.int32)
            self.interior = np.zeros(self.ncells, dtype=bool)
        self.father = None                                        # filled by builder
        self._grid = grid

    def cell_of_vertex(self):
        nx, ny, nz = self._grid.dims
        ax, ay, az = self.axes
        ty, tz = self.shape[1], self.shape[2]
        rx = ax.rank
        ry = ay.rank
        rz = az.rank
        return (rx[None, None, :] * (ty * tz) + ry[None, :, None] * tz
                + rz[:, None, None]).ravel()

    def cell_sizes(self):
        ax, ay, az = self.axes
        wx, wy, wz = (a.hi - a.lo + 1 for a in self.axes)
        return wx[self.cx] * wy[self.cy] * wz[self.cz]

    def cell_vertices(self, cid):
        """Sorted vertex ids of one cell (x fastest)."""
        nx, ny, _ = self._grid.dims
        ax, ay, az = self.axes
        i = np.arange(ax.lo[self.cx[cid]], ax.hi[self.cx[cid]] + 1)
        j = np.arange(ay.lo[self.cy[cid]], ay.hi[self.cy[cid]] + 1)
        k = np.arange(az.lo[self.cz[cid]], az.hi[self.cz[cid]] + 1)
        return (i[None, None, :] + nx * (j[None, :, None] + ny * k[:, None, None])).ravel()

    def vertex_order(self):
        """All vertex ids grouped by cell id (cells ascending, vertices
        ascending within a cell) plus the CSR pointer per cell.

        No sort: a vertex's slot is its cell's start plus its rank inside
        the cell's box (k-major, then j, then i, i.e. ascending vertex id)."""
        nx, ny, nz = self._grid.dims
        ax, ay, az = self.axes
        ptr = np.zeros(self.ncells + 1, dtype=np.int64)
        np.cumsum(self.cell_sizes(), out=ptr[1:])
        ty, tz = self.shape[1], self.shape[2]
        i, j, k = np.arange(nx), np.arange(ny), np.arange(nz)
        wx = (ax.hi - ax.lo + 1)[ax.rank]              # box width of each index's label
        wy = (ay.hi - ay.lo + 1)[ay.rank]
        ox, oy, oz = i - ax.lo[ax.rank], j - ay.lo[ay.rank], k - az.lo[az.rank]
        cell = (ax.rank[None, None, :] * (ty * tz) + ay.rank[None, :, None] * tz + az.rank[:, None, None])
        local = (oz[:, None, None] * wy[None, :, None] + oy[None, :, None]) * wx[None, None, :] + ox[None, None, :]
        slot = (ptr[cell] + local).ravel()
        order = np.empty(nx * ny * nz, dtype=np.int64)
        order[slot] = np.arange(nx * ny * nz, dtype=np.int64)
        return order, ptr


class PartitionHierarchy:
    """Hierarchy of HLevels; `.levels` materialises the reference's
    Level/Cell objects (partition.py:64-98) lazily for API compatibility."""

    def __init__(self, grid, b, kind, hlevels):
        self.grid = grid
        self.b = b
        self.kind = kind
        self.hlevels = hlevels
        self._levels = None

    @property
    def levels(self):
        if self._levels is None:
            out = []
            for t, hl in enumerate(self.hlevels):
                cells = []
                ax, ay, az = hl.axes
                for c in range(hl.ncells):
                    box = ((int(ax.lo[hl.cx[c]]), int(ax.hi[hl.cx[c]])),
                           (int(ay.lo[hl.cy[c]]), int(ay.hi[hl.cy[c]])),
                           (int(az.lo[hl.cz[c]]), int(az.hi[hl.cz[c]])))
                    kc = int(hl.kind_code[c])
                    kind = "general" if kc == 4 else KIND_NAMES[kc]
                    role = "interior" if hl.interior[c] else "separator"
                    cells.append(Cell(c, hl.cell_vertices(c), kind, role, box))
                fa = {} if hl.father is None else {int(c): int(f) for c, f in enumerate(hl.father)}
                out.append(Level(cells=cells, father=fa))
            self._levels = out
        return self._levels

    def to_debug_json(self):
        out = []
        for t, level in enumerate(self.levels):
            out.append({
                "level": t + 1,
                "cells": [{"id": c.id, "size": c.size, "kind": c.kind, "role": c.role,
                           "box": [list(map(int, ex)) for ex in c.box]} for c in level.cells],
                "father": {str(k): v for k, v in sorted(level.father.items())},
            })
        return json.dumps({"b": self.b, "type": self.kind, "levels": out}, indent=1)


def _build(grid, b, nested):
    levels = []
    d = b
    while True:
        hl = HLevel(grid, d, nested)
        if levels:
            prev = levels[-1]
            ux, uy, uz = (prev.axes[a].up(hl.axes[a]) for a in range(3))
            ty, tz = hl.shape[1], hl.shape[2]
            prev.father = (ux[prev.cx] * (ty * tz) + uy[prev.cy] * tz + uz[prev.cz]).astype(np.int64)
        levels.append(hl)
        if hl.ncells == 1:
            return levels
        d *= 2


def build_nested_hierarchy(grid, b):
    """Nested-dissection family (reference partition.py:202-217)."""
    if b <= 1:
        raise ValueError("b must be > 1")
    if all(n < b for n in grid.dims):
        raise GridTooSmallError(f"grid {grid.dims} admits no cutting plane at level 1 with b={b}")
    return PartitionHierarchy(grid, b, "nested", _build(grid, b, True))


def build_general_hierarchy(grid, b):
    """Box-tiling family (reference partition.py:220-229)."""
    if b < 2:
        raise ValueError("b must be >= 2")
    if all(n <= b for n in grid.dims):
        raise GridTooSmallError(f"grid {grid.dims} yields a single box at level 1 with b={b}")
    return PartitionHierarchy(grid, b, "general", _build(grid, b, False))


def expand_to_unknowns(cell, grid):
    """Component-major unknown ids of a cell (reference partition.py:232-242)."""
    nv = grid.n_vertices
    comps = grid.components_per_vertex
    if comps == 1:
        return cell.vertex_ids.copy()
    return np.concatenate([cell.vertex_ids + c * nv for c in range(comps)])


def level1_unknowns(hier):
    """(unknown ids grouped by level-1 cell, CSR pointer): the expansion of
    every level-1 cell (input to the native factorization), computed by the
    native host helper sgf_cell_unknowns (OpenMP over cells)."""
    from . import _native as N

    hl = hier.hlevels[0]
    nx, ny, nz = hier.grid.dims
    tx, ty, tz = hl.shape
    comps = hier.grid.components_per_vertex
    ptr = np.empty(hl.ncells + 1, dtype=np.int64)
    out = np.empty(hier.grid.n_vertices * comps, dtype=np.int64)
    ax, ay, az = hl.axes
    arrs = [np.ascontiguousarray(v, dtype=np.int64) for v in (ax.lo, ax.hi, ay.lo, ay.hi, az.lo, az.hi)]
    st = N.lib().sgf_cell_unknowns(nx, ny, nz, tx, ty, tz, *[a.ctypes.data for a in arrs], comps, ptr.ctypes.data,
                                   out.ctypes.data)
    N.raise_for(st, None, "level-1 cell expansion")
    return out, ptr


def level1_unknowns_numpy(hier):
    """Same as level1_unknowns, in numpy (cross-check in the CPU tests)."""
    hl = hier.hlevels[0]
    verts, vptr = hl.vertex_order()
    comps = hier.grid.components_per_vertex
    if comps == 1:
        return verts, vptr
    nv = hier.grid.n_vertices
    sizes = np.diff(vptr)
    ptr = np.zeros(hl.ncells + 1, dtype=np.int64)
    np.cumsum(sizes * comps, out=ptr[1:])
    out = np.empty(nv * comps, dtype=np.int64)
    # position of vertex slot s (in cell c) for component k: ptr[c] + k*size_c + (s - vptr[c])
    cell_of_slot = np.repeat(np.arange(hl.ncells), sizes)
    local = np.arange(nv) - vptr[cell_of_slot]
    for k in range(comps):
        out[ptr[cell_of_slot] + k * sizes[cell_of_slot] + local] = verts + k * nv
    return out, ptr
