"""Per-factor / per-vector errors of the GPU path against one full-size
reference fixture (tests/golden/*_full.npz, tpfa40_b9.npz), under pivot
replay.  Usage: python tools/full_golden_report.py tpfa40_b9 [--free]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1907_03406_b200 as sgf  # noqa: E402
from conftest import FullGolden  # noqa: E402
from test_full_size_golden import _check_factor  # noqa: E402


def main(name, free=False):
    g = FullGolden(name)
    t = time.time()
    prob = g.problem()
    print(f"[{name}] problem {time.time() - t:.1f}s n={prob.n}", flush=True)
    P = sgf.factorize(prob, replay_perms=None if free else g.perms(), **g.opts)
    print("stats equal:", P.stats == g.stats, " trace equal:",
          [tuple(e) for e in P.rank_trace.entries] == g.trace())
    if P.stats != g.stats:
        for k in g.stats:
            if P.stats.get(k) != g.stats[k]:
                print("  stat differs:", k, str(P.stats.get(k))[:200], "| ref", str(g.stats[k])[:200])
    fac = P.factors
    for k in g["sampled_factors"]:
        k = int(k)
        f = fac[k]
        try:
            e = _check_factor(g, k, f)
            print(f"  f{k:5d} {f.kind:18s} m={f.m:5d} c={f.c:6d} lvl={f.level} "
                  + " ".join(f"{a}={b:.1e}" for a, b in e.items()), flush=True)
        except AssertionError as ex:
            print(f"  f{k:5d} {f.kind} structure mismatch {ex}")
    rhs = g.rhs()
    proj = g.proj()
    for key, op in (("apply_inverse", P.apply_inverse), ("apply_operator", P.apply_operator)):
        y = op(rhs)
        print(f"  {key}: sample/proj/norm rel err", ["%.2e" % v for v in g.vec_errors(key, y, proj)])
        if key in g:
            print(f"  {key}: full rel err %.2e" % (np.linalg.norm(y - g[key]) / np.linalg.norm(g[key])))
    x, rep = sgf.pcg(prob.matrix, rhs, precond=P, tol=1e-12)
    h = np.array(rep.residual_history)
    ref = g["pcg_hist"]
    k = min(len(h), len(ref)) - 1
    if "pcg_hist_alt" in g:
        alt = g["pcg_hist_alt"]
        n = min(k, len(alt) - 1)
        print("  reference's own history spread (A@v vs tril+triu order): max %.2e" %
              np.max(np.abs(alt[:n] - ref[:n]) / ref[:n]))
    from test_full_size_golden import stable_prefix
    print("  1e-10 gate applies to history[0:%d] of %d" % (stable_prefix(g, k), k))
    bad = np.nonzero(np.abs(h[:k] - ref[:k]) > 1e-10 * ref[:k])[0]
    for i in bad[:12]:
        print(f"    history[{i}] gpu {h[i]:.6e} ref {ref[i]:.6e} rel {abs(h[i] - ref[i]) / ref[i]:.2e}")
    print(f"  pcg iters {rep.iterations} (ref {int(g['pcg_iters'])}), max hist rel err "
          f"{np.max(np.abs(h[:k] - ref[:k]) / ref[:k]):.2e}, x errs",
          ["%.2e" % v for v in g.vec_errors("pcg_x", x, proj)])


if __name__ == "__main__":
    main(sys.argv[1], "--free" in sys.argv)
