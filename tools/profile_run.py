"""One factorize + pcg of a config (target for ncu launch lists)."""
import sys
sys.path.insert(0, '.')
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200.problems import CONFIGS, config_rhs
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[cfg]
prob = c["make"]()
P = sgf.factorize(prob, scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
x, rep = sgf.pcg(prob.matrix, config_rhs(prob.n, c["seed"]), precond=P, tol=1e-12)
print("iters", rep.iterations)
