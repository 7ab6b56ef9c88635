"""Asynchronous factorization timeline (SGF_TRACE=3) for a config; Python-side
preamble timed separately."""
import os, sys, time
os.environ["SGF_TRACE"] = sys.argv[2] if len(sys.argv) > 2 else "3"
sys.path.insert(0, '.')
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200.problems import CONFIGS
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
prob = c["make"]()
for rep in range(2):
    t = time.perf_counter()
    P = sgf.factorize(prob, scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
    print("factorize wall %.1f ms" % ((time.perf_counter() - t) * 1e3), flush=True)
    del P
