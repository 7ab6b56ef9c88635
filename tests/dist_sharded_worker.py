"""Worker for the sharded-path tests (launched with torch.distributed.run).

--mode plan   (CPU, gloo): every rank computes the shard plan of a few
              hierarchies; the plans are compared across ranks and checked
              for ownership invariants; the host comm helpers are exercised.
--mode solve  (GPU, gloo or nccl): sharded factorize + apply + PCG against
              the single-GPU path on the same inputs, with the single-GPU
              run's QR pivots replayed (near-tie pivots are not robust to the
              rounding-level reordering of shared Schur sums).
Rank 0 prints one JSON line with the measured differences."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def plan_mode():
    from paper_1907_03406_b200 import sharded as S
    from paper_1907_03406_b200.partition import CartesianGrid, build_nested_hierarchy

    rank, world = dist.get_rank(), dist.get_world_size()
    out = {}
    for dims, b, skip, comp in [((30, 30, 30), 3, 2, True), ((128, 128, 128), 9, 2, True),
                                ((100, 100, 1), 3, 2, True), ((30, 30, 30), 3, 2, False),
                                ((40, 40, 40), 9, 2, True)]:
        hier = build_nested_hierarchy(CartesianGrid(dims=dims), b)
        for nr in (2, 4, 8):
            cr, stop, p = S.shard_plan(hier, nr, skip, comp)
            S.check_plan(hier, cr, stop)
            t = torch.tensor(cr, dtype=torch.int64)
            mx, mn = t.clone(), t.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(mn, op=dist.ReduceOp.MIN)
            assert torch.equal(mx, t) and torch.equal(mn, t), "plans differ across ranks"
            used = sorted(set(int(v) for v in cr if v >= 0))
            out[f"{dims}-{b}-{comp}-{nr}"] = {"stop": stop, "p": p, "ranks_used": used,
                                              "shared": int((cr < 0).sum()), "cells": int(cr.size)}
    # comm helpers on CPU tensors
    v = torch.full((5,), float(rank + 1), dtype=torch.float64)
    S._reduce_sum(v)
    w = torch.full((3,), float(rank + 7), dtype=torch.float64)
    S._broadcast(w)
    z = torch.zeros(world, dtype=torch.float64)
    z[rank] = rank + 0.5
    S._allreduce_sum(z)
    out["reduce"] = v.tolist() if rank == 0 else None
    out["bcast"] = w.tolist()
    out["allreduce"] = z.tolist()
    return out


def solve_mode(args):
    import paper_1907_03406_b200 as sgf
    from paper_1907_03406_b200 import problems as PB
    from paper_1907_03406_b200 import sharded as S

    rank = dist.get_rank()
    dev = int(os.environ.get("LOCAL_RANK", "0")) if args.per_rank_gpu else 0
    torch.cuda.set_device(dev)
    res = {}
    cases = {
        "p3d30_b3": (lambda: PB.poisson7(30, spacing=1.0 / 31), dict(scheme="nest-2-2", degree=1, b=3, rank_tol=1e-2)),
        "aniso26_b3": (lambda: PB.anisotropic7(26), dict(scheme="nest-2-2", degree=1, b=3, rank_tol=1e-3)),
        "p2d100_b3": (lambda: PB.poisson2d(100), dict(scheme="nest-2-2", degree=1, b=3, rank_tol=1e-2)),
        "p3d30_exact": (lambda: PB.poisson7(30, spacing=1.0 / 31), dict(scheme="nest-2-2", degree=1, b=3,
                                                                           mode="exact")),
        "elast8_b3": (lambda: PB.elasticity_cube(8), dict(scheme="nest-2-2", degree=1, b=3, rank_tol=1e-2)),
        # BASELINE config 2: level-3 nodes of 2654-3571 unknowns take the
        # INT8-emulated products and the recursive Cholesky
        "cfg2": (PB.CONFIGS[2]["make"], dict(scheme="nest-2-2", degree=1, b=9, rank_tol=1e-2)),
    }
    def note(msg):
        if args.verbose:
            print(f"[rank {rank}] {msg}", file=sys.stderr, flush=True)

    for name in args.cases.split(","):
        make, opts = cases[name]
        note(f"case {name}")
        prob = make()
        n = prob.matrix.shape[0]
        rhs = np.random.default_rng(3).uniform(-1, 1, n)
        # single-GPU reference on every rank (identical inputs -> identical result)
        P1 = sgf.factorize(prob, device=dev, **opts)
        perms = [np.asarray(f.perm) for f in P1.factors if f.kind == "CompressionFactor"]
        y1 = P1.apply_inverse(rhs)
        x1, rep1 = sgf.pcg(sgf.DeviceCSR(prob.matrix, device=dev), rhs, precond=P1, tol=1e-12)
        note("single-GPU path done")
        PS = S.factorize_sharded(prob, device=dev, replay_perms=perms, **opts)
        note("sharded factorization done")
        ys = PS.apply_inverse(rhs)
        note("sharded apply done")
        xs, reps = S.pcg_sharded(sgf.DeviceCSR(prob.matrix, device=dev), rhs, PS, tol=1e-12)
        r = {
            "n": n,
            "apply_rel": float(np.linalg.norm(ys - y1) / np.linalg.norm(y1)),
            "x_rel": float(np.linalg.norm(xs - x1) / np.linalg.norm(x1)),
            "iters": [rep1.iterations, reps.iterations],
            "hist_rel": float(max(abs(a - b) / max(abs(b), 1e-300) for a, b in
                                  zip(reps.residual_history[:-1], rep1.residual_history[:-1]))) if
            len(rep1.residual_history) > 1 else 0.0,
            "local_factors": PS.n_local_factors,
            "local_levels": sorted({f.level for f in PS.pre.factors[:PS.n_local_factors]}),
            "local_big": sum(1 for f in PS.pre.factors[:PS.n_local_factors] if f.m >= 1024),
            "top_unknowns": int(len(PS.top_idx)),
            "stop": PS.plan.get("stop"),
            "partition_level": PS.plan.get("partition_level"),
        }
        log = PS.exchange_log
        if log:
            meta = np.asarray(log["sent_meta"]).reshape(-1, 4)
            # a rank != 0 sends only blocks touching its own cells, or shared
            # (top-separator x top-separator) blocks carrying its Schur sums
            if rank != 0 and len(meta):
                ok = (meta[:, 2] == rank) | (meta[:, 3] == rank) | ((meta[:, 2] < 0) & (meta[:, 3] < 0))
            else:
                ok = np.ones(len(meta), bool)
            r.update(exchange_blocks=int(log["nblocks"]), sent_blocks=int(log["sent_blocks"]),
                     sent_bytes=int(log["sent_bytes"]), exchange_ok=bool(ok.all()),
                     sent_foreign=int((~ok).sum()), per_rank=log["per_rank"])
        if args.free:
            # free-running pivots: iteration count within +-1 (SURVEY.md 8c gate 5)
            PF = S.factorize_sharded(prob, device=dev, **opts)
            _, repf = S.pcg_sharded(sgf.DeviceCSR(prob.matrix, device=dev), rhs, PF, tol=1e-12)
            r["iters_free"] = repf.iterations
            r["converged_free"] = bool(repf.converged)
            del PF
        if args.debug:
            # compare this rank's factors with the single-GPU factors of the same (level, node, type)
            key1 = {(f.level, f.node, f.kind): f for f in P1.factors}
            bad = []
            for k, f in enumerate(PS.pre.factors):
                g = key1.get((f.level, f.node, f.kind))
                if g is None:
                    bad.append((k, f.level, f.node, f.kind, "missing"))
                    continue
                d = float(np.max(np.abs(f.L - g.L))) if f.L.shape == g.L.shape else -1.0
                if d > 1e-8 * max(1.0, float(np.max(np.abs(g.L)))):
                    bad.append((k, f.level, f.node, f.kind, d))
            r["factor_mismatch"] = bad[:8]
            r["n_mismatch"] = len(bad)
        if rank == 0:
            keys = ("flops_factorize", "flops_apply", "peak_blocks_bytes", "factors", "per_level",
                    "final_dense_size", "max_node_size")
            r["stats_equal"] = all(PS.stats[k] == P1.stats[k] for k in keys)
            r["stats_diff"] = [k for k in keys if PS.stats[k] != P1.stats[k]]
            r["trace_equal"] = PS.rank_trace == P1.rank_trace
        res[name] = r
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="plan")
    ap.add_argument("--backend", default="gloo")
    ap.add_argument("--cases", default="p3d30_b3")
    ap.add_argument("--per-rank-gpu", action="store_true")
    ap.add_argument("--debug", action="store_true")
    ap.add_argument("--free", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--dump-after", type=float, default=0.0,
                    help="print every thread's Python stack to stderr after this many seconds (hang diagnosis)")
    args = ap.parse_args()
    if args.dump_after > 0:
        import faulthandler
        faulthandler.dump_traceback_later(args.dump_after, exit=False)
    dist.init_process_group(backend=args.backend)
    try:
        out = plan_mode() if args.mode == "plan" else solve_mode(args)
        gathered = [None] * dist.get_world_size()
        dist.all_gather_object(gathered, out)
        if dist.get_rank() == 0:
            print("RESULT " + json.dumps({"world": dist.get_world_size(), "ranks": gathered}))
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
