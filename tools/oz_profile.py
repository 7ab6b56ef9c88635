"""Cycle breakdown of the INT8-emulated products over one cfg-N factorization
(OZ_PROFILE build of libsgf.so in build/oz_prof/, made by this script):
MMA thread waiting for operands / for the epilogue / issuing, epilogue
draining / waiting for the MMAs, summed over CTAs."""
import ctypes as C
import os
import subprocess
import sys

sys.path.insert(0, '.')
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(ROOT, "build", "oz_prof")
lib = os.path.join(out, "libsgf.so")
if not os.path.exists(lib):
    raise SystemExit("build first: make -C paper_1907_03406_b200/csrc OZPROF=1 (see tools/oz_profile.sh)")
from paper_1907_03406_b200 import _native as N
N.load_library(lib)
import paper_1907_03406_b200 as sgf
from paper_1907_03406_b200.problems import CONFIGS
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
prob = c["make"]()
L = C.CDLL(lib)
buf = (C.c_ulonglong * 8)()
for rep in range(2):
    L.sgf_oz_prof_read(buf, 1)
    P = sgf.factorize(prob, scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"])
    N.lib().sgf_sync(P._ctx)
    L.sgf_oz_prof_read(buf, 1)
    del P
names = ["mma_wait_operands", "mma_wait_epilogue", "mma_issue", "epi_drain", "epi_wait_mma"]
tot = sum(buf[i] for i in range(3))
print({n: buf[i] for i, n in enumerate(names)})
print({n: round(buf[i] / max(tot, 1), 3) for i, n in enumerate(names[:3])}, "(fractions of the MMA thread's time)")
