"""First apply of a fresh preconditioner (CUDA-graph capture + instantiate of
the sweeps) against later applies, cfg 4."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200.problems import CONFIGS, config_rhs
c = CONFIGS[4]; prob = c["make"](); rhs = config_rhs(prob.n, c["seed"])
r = torch.tensor(rhs, device="cuda")
for rep in range(3):
    P = sgf.factorize(prob, scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
    torch.cuda.synchronize()
    ts = []
    for k in range(3):
        t = time.perf_counter(); y = P.apply_inverse(r); torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
    print("apply ms: first %.1f, then %.1f %.1f" % tuple(ts), flush=True)
    del P
