import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200.problems import CONFIGS, config_rhs
c = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]; prob = c["make"](); rhs = config_rhs(prob.n, c["seed"])
P = sgf.factorize(prob, scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
for rep in range(3):
    t = time.perf_counter(); A = sgf.DeviceCSR(prob.matrix); t1 = time.perf_counter()
    x, r = sgf.pcg(A, rhs, precond=P, tol=1e-12); t2 = time.perf_counter()
    x, r = sgf.pcg(prob.matrix, rhs, precond=P, tol=1e-12); t3 = time.perf_counter()
    print("csr %.1f ms  pcg(DeviceCSR) %.1f ms  pcg(scipy) %.1f ms" % ((t1-t)*1e3, (t2-t1)*1e3, (t3-t2)*1e3), flush=True)
