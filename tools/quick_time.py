"""Quick timing of factorize + pcg for a BASELINE config (dev tool)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200.problems import CONFIGS, config_rhs

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[cfg]
t = time.perf_counter(); prob = c["make"](); tg = time.perf_counter() - t
rhs = config_rhs(prob.n, c["seed"])
for rep in range(2):
    t = time.perf_counter()
    P = sgf.factorize(prob, scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
    tf = time.perf_counter() - t
    t = time.perf_counter()
    x, r = sgf.pcg(prob.matrix, rhs, precond=P, tol=1e-12)
    ts = time.perf_counter() - t
    print(json.dumps(dict(cfg=cfg, n=prob.n, t_gen=tg, t_F=tf, t_S=ts, iters=r.iterations,
                          final=r.final_rel_residual, flops=P.stats["flops_factorize"],
                          tflops=P.stats["flops_factorize"] / tf / 1e12, ranks=[len(l["ranks"]) for l in P.stats["per_level"]])), flush=True)
    del P
