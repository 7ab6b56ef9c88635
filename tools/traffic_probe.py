"""Algorithmic bytes of the apply's level-3 coupling and inverse sweeps (cfg4),
to pair with the ncu dram byte count of the same launches
(profiles/ncu_traffic.json): per level, E dense (8 c m), E nonzero 32-column
tiles, and the same for the L^{-1} triangles that carry tile masks."""
import ctypes as C
import json
import sys

import numpy as np

sys.path.insert(0, '.')
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200 import _native as N
from paper_1907_03406_b200.problems import CONFIGS

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
P = sgf.factorize(c["make"](), scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
out = {}
for lev in sorted({f.level for f in P.factors if f.kind == "EliminationFactor"}):
    e_dense = sum(8 * f.c * f.m for f in P.factors if f.kind == "EliminationFactor" and f.level == lev)
    buf = np.zeros(2)
    N.raise_for(N.lib().sgf_precond_coupling_bytes_level(P._h, lev, buf.ctypes.data), P._ctx)
    out[lev] = {"E_dense": e_dense, "E_and_masked_Linv_dense": buf[0], "E_and_masked_Linv_nonzero": buf[1]}
print(json.dumps(out))
det = {}
for lev in sorted({f.level for f in P.factors if f.kind == "EliminationFactor"}):
    buf = np.zeros(6)
    N.raise_for(N.lib().sgf_precond_coupling_bytes_detail(P._h, lev, buf.ctypes.data), P._ctx)
    det[lev] = dict(zip(("dense", "nonzero_tiles", "from_first_tile", "chunks256", "chunks256_trimmed", "tile_runs"),
                        (float(v) for v in buf)))
print(json.dumps({"forward_sweep_E_bytes": det}))
