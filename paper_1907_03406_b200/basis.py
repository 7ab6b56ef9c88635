"""Polynomial basis Pi over vertex coordinates (reference `basis.py:15-62`).

Columns [1, x, y, z (, x^2, y^2, z^2, xy, yz, zx)], replicated block
diagonally per component under component-major unknown ordering, each
column scaled to unit max-norm (zero columns left as they are).
"""

from dataclasses import dataclass

import numpy as np

PI_COLS_SCALAR = {0: 1, 1: 4, 2: 10}


@dataclass
class PolyBasis:
    Pi: np.ndarray
    degree: int
    pi_cols: int


def build_polynomial_basis(coords, degree, components=1):
    coords = np.asarray(coords, dtype=float)
    if degree not in (0, 1, 2):
        raise ValueError(f"degree must be 0, 1, or 2, got {degree}")
    if components not in (1, 3):
        raise ValueError(f"components must be 1 or 3, got {components}")
    nv = len(coords)
    ps = PI_COLS_SCALAR[degree]
    # scalar block S (nv x ps), every column divided by its max |entry|
    # (zero columns stay); replicated blocks share the scalar column's scale
    S = np.empty((nv, ps))
    S[:, 0] = 1.0
    if degree >= 1:
        S[:, 1:4] = coords
    if degree >= 2:
        x, y, z = coords[:, 0], coords[:, 1], coords[:, 2]
        S[:, 4], S[:, 5], S[:, 6] = x * x, y * y, z * z
        S[:, 7], S[:, 8], S[:, 9] = x * y, y * z, z * x
    if nv and ps > 1:
        s = np.maximum(S[:, 1:].max(axis=0), -S[:, 1:].min(axis=0))
        s[s == 0] = 1.0
        S[:, 1:] /= s
    if components == 1:
        Pi = S
    else:
        Pi = np.zeros((components * nv, components * ps))
        for c in range(components):
            Pi[c * nv:(c + 1) * nv, c * ps:(c + 1) * ps] = S
    return PolyBasis(Pi=Pi, degree=degree, pi_cols=Pi.shape[1])
