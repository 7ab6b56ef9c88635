"""factorize cfg N twice; the second one inside cudaProfilerStart/Stop
(ncu --profile-from-start off target: per-launch list of one factorization)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200.problems import CONFIGS
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
prob = c["make"]()
P = sgf.factorize(prob, scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
del P
torch.cuda.synchronize()
torch.cuda.profiler.start()
P = sgf.factorize(prob, scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
