"""Time apply_inverse and pcg on a factorized config (device-resident vectors)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200.problems import CONFIGS, config_rhs
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
prob = c["make"]()
P = sgf.factorize(prob, scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
r = torch.tensor(config_rhs(prob.n, c["seed"]), device="cuda")
torch.cuda.synchronize()
for _ in range(3):
    y = P.apply_inverse(r)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    y = P.apply_inverse(r)
torch.cuda.synchronize()
ta = (time.perf_counter() - t) / 20
A = sgf.DeviceCSR(prob.matrix)
x, rep = sgf.pcg(A, r, precond=P, tol=1e-12)
t = time.perf_counter()
x, rep = sgf.pcg(A, r, precond=P, tol=1e-12)
ts = time.perf_counter() - t
print(json.dumps({"apply_ms": ta * 1e3, "pcg_s": ts, "iters": rep.iterations, "per_iter_ms": ts / rep.iterations * 1e3}))
