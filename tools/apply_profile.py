"""factorize cfg N, then two apply_inverse calls (ncu target for the apply kernels)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200.problems import CONFIGS, config_rhs
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
prob = c["make"]()
P = sgf.factorize(prob, scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
r = config_rhs(prob.n, c["seed"])
for _ in range(2):
    y = P.apply_inverse(r)
print("ok", float(np.linalg.norm(y)))
