"""Host/device phase breakdown of one factorize + pcg (SGF_TRACE=1)."""
import os, sys, time
os.environ["SGF_TRACE"] = "1"
sys.path.insert(0, '.')
import numpy as np
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200 import partition as Pm, basis as Bm
from paper_1907_03406_b200.problems import CONFIGS, config_rhs
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
prob = c["make"]()
opts = dict(scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
P = sgf.factorize(prob, **opts); del P
t = time.perf_counter(); H = Pm.build_nested_hierarchy(prob.grid, c["b"]); print("hier %.3f" % (time.perf_counter() - t))
t = time.perf_counter(); u = Pm.level1_unknowns(H); print("l1unk %.3f" % (time.perf_counter() - t))
t = time.perf_counter(); B = Bm.build_polynomial_basis(prob.coords, 1, prob.grid.components_per_vertex); print("basis %.3f" % (time.perf_counter() - t))
t = time.perf_counter(); A = prob.matrix.tocsr(); print("tocsr %.3f sorted=%s" % (time.perf_counter() - t, A.has_sorted_indices))
sys.stderr.flush()
t = time.perf_counter()
P = sgf.factorize(prob, **opts)
print("factorize total %.3f" % (time.perf_counter() - t), flush=True)
rhs = config_rhs(prob.n, c["seed"])
t = time.perf_counter(); x, rep = sgf.pcg(prob.matrix, rhs, precond=P, tol=1e-12); print("pcg %.3f it %d" % (time.perf_counter() - t, rep.iterations))
