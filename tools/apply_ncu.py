"""factorize cfg N, then one apply_inverse inside cudaProfilerStart/Stop
(ncu --profile-from-start off target: per-launch list of one apply)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200.problems import CONFIGS, config_rhs
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
prob = c["make"]()
P = sgf.factorize(prob, scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
r = config_rhs(prob.n, c["seed"])
y = P.apply_inverse(r)
torch.cuda.synchronize()
torch.cuda.profiler.start()
y = P.apply_inverse(r)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", float(np.linalg.norm(y)))
