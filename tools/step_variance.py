"""Per-step factor / solve device times of the bench's device-resident step
(cfg 4), to look at step-to-step variance."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200 import _native as N
from paper_1907_03406_b200.problems import CONFIGS, config_rhs
c = CONFIGS[4]; prob = c["make"](); A = prob.matrix.tocsr(); A.sort_indices()
rhs = config_rhs(prob.n, c["seed"])
vals = torch.tensor(A.data, device="cuda"); ip = torch.tensor(A.indptr, dtype=torch.int64, device="cuda")
ix = torch.tensor(A.indices, dtype=torch.int32, device="cuda"); b = torch.tensor(rhs, device="cuda")
Ad = sgf.DeviceCSR(device=0, indptr=ip, indices=ix, values=vals, n=prob.n)
st = torch.cuda.ExternalStream(N.lib().sgf_stream(N.context(0)))
opts = dict(scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(st)
    P = sgf.factorize(prob, device_values=vals, **opts)
    e[1].record(st)
    x, rep = sgf.pcg(Ad, b, precond=P, tol=1e-12)
    e[2].record(st)
    torch.cuda.synchronize()
    print("step %d factor %.1f ms solve %.1f ms iters %d" % (k, e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), rep.iterations), flush=True)
    del P
