"""GPU: every alternative kernel path the library selects by shape (or that an
environment switch forces) meets the same parity gates as the default path.

Each variant runs in a subprocess (the switches are read once per process):
BASELINE config 2 (3-D Poisson 64^3, b = 9) exercises the level-1 sparse
eliminations, the INT8-emulated level-2 Schur updates and level-3 products,
the recursive Cholesky, the shared-memory QR, the banded level-1 sweeps and
the bulk-copy apply kernels, so each switch below replaces a kernel that the default run uses.
Gates as in test_gpu_parity.py: stats and rank trace bit-exact, apply
within 1e-10 of the reference under pivot replay, PCG iterations equal."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = {
    "default": {},
    "l1_dense_g": {"SGF_L1_BAND": "0"},                # level-1 sweeps through the dense G = A_BB^-1 (bulk-copy symv)
    "symv_registers": {"SGF_SYMV": "0", "SGF_L1_BAND": "0"},  # ... with the register-staged symmetric GEMV
    "gemv_no_bulk": {"SGF_GEMV_BULK": "0"},            # 32-lane GEMV for the long rows too
    "gemv_sparse_ring": {"SGF_GEMV_SPARSE_RING": "1"},  # block-sparse rows through the bulk-copy ring (not tile lists)
    "qr_l2_panel": {"SGF_QR_SMEM": "0"},               # cluster QR with the panel in L2
    "qr_l2_panel_8x1024": {"SGF_QR_SMEM": "0", "SGF_QR_CL": "81024"},  # ... on portable 8-CTA clusters
    "qr_l2_panel_16x256": {"SGF_QR_SMEM": "0", "SGF_QR_CL": "160256"},  # ... with 256-thread CTAs
    "qr_cluster16": {"SGF_QR_SMEM": "16"},             # shared-memory QR forced to 16-CTA clusters
    "l1_dense": {"SGF_NO_L1SPARSE": "1"},              # level-1 E and Schur as dense DMMA GEMMs
    "l1_e_eager": {"SGF_L1E_EAGER": "1"},              # level-1 couplings E formed during the factorization
    "diag_left_looking": {"SGF_DIAG_CHOL": "0"},       # left-looking 64x64 diagonal Cholesky
    "diag_shared_rl": {"SGF_DIAG_CHOL": "1"},          # right-looking diagonal Cholesky in shared memory
    "split_warp": {"SGF_OZ_SPLIT_WARP": "1"},          # warp-per-group operand split
    "l2_schur_dmma": {"SGF_OZAKI_SCHUR_MIN_M": "0"},   # level-2 Schur on DMMA
    "no_emulation": {"SGF_OZAKI_MIN_M": "0"},          # every product on DMMA
}

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %(root)r)
sys.path.insert(0, %(tests)r)
import paper_1907_03406_b200 as sgf
from conftest import Golden
from paper_1907_03406_b200.problems import CONFIGS, config_rhs
g = Golden("cfg2")
prob = CONFIGS[2]["make"]()
P = sgf.factorize(prob, replay_perms=g.perms(), **g.opts)
rhs = config_rhs(prob.n, 1)
y = P.apply_inverse(rhs)
err = float(np.linalg.norm(y - g["apply_inverse"]) / np.linalg.norm(g["apply_inverse"]))
x, rep = sgf.pcg(prob.matrix, rhs, precond=P, tol=1e-12)
print(json.dumps({"stats_equal": P.stats == g.stats,
                  "trace_equal": [tuple(e) for e in P.rank_trace.entries] == g.trace(),
                  "apply_err": err, "iters": rep.iterations, "ref_iters": int(g["pcg_iters"])}))
"""


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_parity(name):
    env = dict(os.environ)
    env.update(VARIANTS[name])
    code = SCRIPT % {"root": ROOT, "tests": os.path.join(ROOT, "tests")}
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["stats_equal"] and res["trace_equal"], res
    assert res["apply_err"] <= 1e-10, res
    assert res["iters"] == res["ref_iters"], res
