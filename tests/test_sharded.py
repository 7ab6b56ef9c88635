"""Sharded (multi-rank) path, SURVEY.md 8e.

CPU: two gloo ranks compute the shard plan (ownership of level-1 cells) for
several hierarchies and must agree; ownership invariants hold; the comm
helpers reduce / broadcast / all-reduce correctly.

GPU: two ranks sharing the one GPU (gloo collectives staged through the
host; no kernel waits on another rank's kernel) run the sharded
factorize -> apply -> PCG and are compared with the single-GPU path on the
same inputs, the single-GPU run's QR pivots replayed."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "dist_sharded_worker.py")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _launch(nproc, *args, timeout=900):
    if "solve" in args:
        # the workers share this session's GPU: hand back what earlier tests
        # left in the allocators' caches (tens of GB after the full-size cases)
        import gc

        import torch

        from paper_1907_03406_b200 import _native as N

        gc.collect()
        free0 = torch.cuda.mem_get_info()[0]
        N.trim_memory()
        torch.cuda.empty_cache()
        print(f"[sharded] free HBM before the workers: {free0 / 2**30:.1f} -> "
              f"{torch.cuda.mem_get_info()[0] / 2**30:.1f} GiB")
        # a hung rank prints its Python stacks before the timeout kills it
        args = (*args, "--verbose", "--dump-after", str(max(60, timeout - 120)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", WORKER, *args]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    except subprocess.TimeoutExpired as e:
        err = e.stderr.decode("utf-8", "replace") if isinstance(e.stderr, bytes) else (e.stderr or "")
        raise AssertionError(f"sharded workers timed out after {timeout} s; stderr tail:\n{err[-6000:]}") from None
    lines = [l for l in out.stdout.splitlines() if l.startswith("RESULT ")]
    assert out.returncode == 0 and lines, out.stdout[-3000:] + out.stderr[-3000:]
    return json.loads(lines[-1][len("RESULT "):])


def test_shard_plan_two_ranks_gloo():
    res = _launch(2, "--mode", "plan", timeout=600)
    assert res["world"] == 2
    r0, r1 = res["ranks"]
    for k in r0:
        if k in ("reduce", "bcast", "allreduce"):
            continue
        assert r0[k] == r1[k]
    assert r0["(128, 128, 128)-9-True-8"] == {"stop": 3, "p": 4, "ranks_used": list(range(8)), "shared": 2437,
                                              "cells": 24389}
    # cfg2-like (3 levels): the level-3 interiors are the partition cells, so
    # their eliminations (the big nodes) run on their owners
    assert r0["(40, 40, 40)-9-True-2"]["stop"] == 3 and r0["(40, 40, 40)-9-True-2"]["p"] == 3
    assert r0["reduce"] == [3.0] * 5 and r1["reduce"] is None
    assert r0["bcast"] == r1["bcast"] == [7.0] * 3
    assert r0["allreduce"] == r1["allreduce"] == [0.5, 1.5]


def _check_solve(res, cases):
    for rk in res["ranks"]:
        for name in cases:
            r = rk[name]
            assert r["apply_rel"] <= 1e-10, (name, r)
            assert r["x_rel"] <= 1e-8, (name, r)
            assert abs(r["iters"][0] - r["iters"][1]) <= 1, (name, r)
            assert r["hist_rel"] <= 1e-8, (name, r)
    for name in cases:
        r = res["ranks"][0][name]
        assert r["stats_equal"], (name, r["stats_diff"])
        assert r["trace_equal"], name
        # the exchange moves only what each rank holds: its own cells' blocks and
        # its partial sums of shared blocks, never another rank's blocks
        for rk in res["ranks"]:
            if "exchange_ok" in rk[name]:
                assert rk[name]["exchange_ok"], (name, rk[name]["sent_foreign"])


@pytest.mark.gpu
def test_sharded_two_ranks_one_gpu():
    cases = ["p3d30_b3", "aniso26_b3", "p2d100_b3", "p3d30_exact", "elast8_b3"]
    res = _launch(2, "--mode", "solve", "--backend", "gloo", "--cases", ",".join(cases), "--free")
    assert res["world"] == 2
    _check_solve(res, cases)
    for name in cases:
        r = res["ranks"][0][name]
        assert r["converged_free"] and abs(r["iters_free"] - r["iters"][0]) <= 1, (name, r)
    # both ranks own work in the local phase
    assert all(rk["p3d30_b3"]["local_factors"] > 0 for rk in res["ranks"])


@pytest.mark.gpu
def test_sharded_single_rank_matches():
    res = _launch(1, "--mode", "solve", "--backend", "gloo", "--cases", "p3d30_b3")
    _check_solve(res, ["p3d30_b3"])


@pytest.mark.gpu
def test_sharded_three_ranks_uneven():
    # 8 octants over 3 ranks (3/3/2): uneven ownership, shared blocks summed from three ranks
    cases = ["p3d30_b3", "aniso26_b3"]
    res = _launch(3, "--mode", "solve", "--backend", "gloo", "--cases", ",".join(cases))
    assert res["world"] == 3
    _check_solve(res, cases)
    assert all(rk["p3d30_b3"]["local_factors"] > 0 for rk in res["ranks"])


@pytest.mark.gpu
def test_sharded_nccl_backend_single_rank():
    # the NCCL code path of the collectives (device buffers, library stream
    # wrapped as the torch stream) with the one GPU this run has
    res = _launch(1, "--mode", "solve", "--backend", "nccl", "--cases", "p3d30_b3")
    _check_solve(res, ["p3d30_b3"])


@pytest.mark.gpu
def test_sharded_cfg2_two_ranks():
    # BASELINE config 2 at full size over two ranks: the large level-3 nodes
    # run the INT8-emulated products inside the rank-local phase / on rank 0
    res = _launch(2, "--mode", "solve", "--backend", "gloo", "--cases", "cfg2", timeout=1500)
    _check_solve(res, ["cfg2"])
    # the level-3 eliminations (2654-3571 unknowns, 71.5% of the flops) run
    # on their owners: 4 on each rank
    for rk in res["ranks"]:
        r = rk["cfg2"]
        assert r["stop"] == 3 and 3 in r["local_levels"], r
        assert r["local_big"] == 4, r
    # rank 1 sends only part of the trailing matrix
    r1 = res["ranks"][1]["cfg2"]
    assert 0 < r1["sent_blocks"] < r1["exchange_blocks"], r1
