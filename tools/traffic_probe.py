"""Algorithmic bytes of the apply's L3 coupling GEMV launch (cfg4), to pair with
the ncu dram byte count of the same launch (profiles/ncu_traffic.json)."""
import sys, json
sys.path.insert(0, '.')
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200.problems import CONFIGS
c = CONFIGS[4]
P = sgf.factorize(c["make"](), scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
by = {}
for f in P.factors:
    if f.kind == "EliminationFactor":
        by.setdefault(f.level, 0)
        by[f.level] += 8 * f.c * f.m
print(json.dumps({"E_bytes_by_level": by}))
