"""A/B timing of the bench step (factorize + pcg, inputs resident) for one
config: `SGF_LIB=<lib> python tools/ab_time.py [cfg] [reps]` prints the median
factor / solve / step times over reps after two warm-up steps.  Pair with
tools/ab_build.sh to time an older revision's library on the same box."""
import os, sys, statistics
sys.path.insert(0, '.')
import torch
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200 import _native as N
from paper_1907_03406_b200.problems import CONFIGS, config_rhs
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
c = CONFIGS[cfg]
prob = c["make"]()
A = prob.matrix.tocsr()
A.sort_indices()
rhs = config_rhs(prob.n, c["seed"])
vals = torch.tensor(A.data, dtype=torch.float64, device="cuda")
ip = torch.tensor(A.indptr, dtype=torch.int64, device="cuda")
ix = torch.tensor(A.indices, dtype=torch.int32, device="cuda")
b_dev = torch.tensor(rhs, dtype=torch.float64, device="cuda")
Ad = sgf.DeviceCSR(device=0, indptr=ip, indices=ix, values=vals, n=prob.n)
stream = torch.cuda.ExternalStream(N.lib().sgf_stream(N.context(0)))
opts = dict(scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"], device=0)


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


tf, ts = [], []
for r in range(reps + 2):
    torch.cuda.synchronize()
    e0 = ev()
    P = sgf.factorize(prob, device_values=vals, **opts)
    e1 = ev()
    x, rep = sgf.pcg(Ad, b_dev, precond=P, tol=1e-12)
    e2 = ev()
    torch.cuda.synchronize()
    del P
    if r >= 2:
        tf.append(e0.elapsed_time(e1))
        ts.append(e1.elapsed_time(e2))
print("lib %s cfg%d: factor %.1f ms (min %.1f) solve %.1f ms (min %.1f) step %.1f ms iters %d" % (
    os.environ.get("SGF_LIB", "in-tree"), cfg, statistics.median(tf), min(tf), statistics.median(ts), min(ts),
    statistics.median([a + b for a, b in zip(tf, ts)]), rep.iterations), flush=True)
