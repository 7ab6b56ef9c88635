"""Solve-phase timing on a config: apply_inverse alone, PCG with the
preconditioner, PCG without (identity), each by wall clock and CUDA events on
the library stream."""
import json
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_1907_03406_b200 as sgf  # noqa: E402
from paper_1907_03406_b200 import _native as N  # noqa: E402
from paper_1907_03406_b200.problems import CONFIGS, config_rhs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
prob = c["make"]()
P = sgf.factorize(prob, scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
r = torch.tensor(config_rhs(prob.n, c["seed"]), device="cuda")
A = sgf.DeviceCSR(prob.matrix)
stream = torch.cuda.ExternalStream(N.lib().sgf_stream(N.context(0)))


def timed(fn, reps=1):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    e0.record(stream)
    for _ in range(reps):
        out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3, e0.elapsed_time(e1) / reps, out


for _ in range(3):
    P.apply_inverse(r)
res = {}
res["apply_wall_ms"], res["apply_event_ms"], _ = timed(lambda: P.apply_inverse(r), 20)
sgf.pcg(A, r, precond=P, tol=1e-12)
w, e, (x, rep) = timed(lambda: sgf.pcg(A, r, precond=P, tol=1e-12))
res.update(pcg_wall_ms=w, pcg_event_ms=e, iters=rep.iterations, per_iter_wall_ms=w / rep.iterations)
w, e, (x, rep) = timed(lambda: sgf.pcg(A, r, precond=None, tol=1e-12, maxit=200))
res.update(cg_wall_ms=w, cg_event_ms=e, cg_iters=rep.iterations, cg_per_iter_ms=w / rep.iterations)
print(json.dumps(res))
