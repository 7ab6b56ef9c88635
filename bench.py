#!/usr/bin/env python
"""Benchmark of the factorize -> PCG hot path (BASELINE.json metric:
"factor+solve wall time & FP64 TFLOP/s on 128^3 Laplace; PCG iters vs CPU ref").

Workload (one step): BASELINE config 4, the 3-D anisotropic Laplace operator
diag(1, 1, 1e-3) on a 128^3 grid (n = 2,097,152, 7-point, float64), nest-2-2,
degree 1, b = 9, rank_tol 1e-3: `factorize` followed by `pcg` to rtol 1e-12
from a zero guess with RHS uniform[-1,1] (seed 4).  Synthetic input of the
exact BASELINE shape (no dataset involved).

  value  factor+solve seconds per step with the CSR values and the RHS already
         resident in HBM (device timed with CUDA events on the library stream);
  e2e    the same step through the public API with host numpy inputs
         (host CSR + RHS in, solution x back on the host), copies included.

Beside the headline the line carries, per BASELINE config cfg1..cfg5
(`configs`): t_F, t_S, PCG iterations against the reference's, ms per
apply_inverse and its GB/s, FP64 TFLOP/s over the factorization; and the
headline step with every FP64 product on IEEE DMMA (`ieee_fp64`: the INT8
emulation switched off).

CPU reference (never extrapolated): `--impl reference` runs the reference
package itself (oracle/_ref, built from /root/reference by
oracle/build_ref.sh) on the full cfg4 problem, one factorize + pcg with one
BLAS thread, timed as the reference's own harness does (reference
bench.py:157-166); the GPU arm's `cpu_baseline` is a bounded sample (the
same package and operator at 40^3 with every host core as BLAS threads,
after the GPU measurements; `--cpu-baseline full` runs the whole cfg4
problem instead, ~15 min).

Run:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sgf|reference]
N > 1 (torchrun, NCCL): the one 128^3 problem is sharded across the ranks
(sharded.py: subtree ownership of the nested-dissection tree, rank-local
elimination phase, the ranks' nonzero trailing blocks summed onto rank 0,
distributed-vector PCG with halo-exchange SpMV and the staged sharded
apply); strong scaling, the step time is the max over ranks.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

# torchrun sets OMP_NUM_THREADS=1 per rank; the native host pipeline (block
# discovery, staging copies, task lists) is OpenMP-parallel, so give each
# rank its share of the host cores instead (before any OpenMP runtime loads)
# (the reference arm runs on rank 0 alone and takes every host core)
if "LOCAL_WORLD_SIZE" in os.environ and os.environ.get("OMP_NUM_THREADS") == "1":
    _ref_arm = "reference" in sys.argv[1:] and "--impl" in sys.argv[1:]
    _share = 1 if _ref_arm else max(1, int(os.environ["LOCAL_WORLD_SIZE"]))
    os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or 1) // _share))

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = 4
FP64_PEAK_TFLOPS = 37.1  # measured DMMA issue rate on this pool's B200 (profiles/fp64_peak_r01.jsonl)
INT8_PEAK_TOPS = 4500.0  # B200 dense INT8 tensor peak (nominal; MEASURED_PEAKS.json has no INT8 figure)
INT8_PEAK_SOURCE = "nominal B200 dense INT8 (4.5 POPS); MEASURED_PEAKS.json has no INT8 figure"
METRIC = "factor+solve wall time (cfg4: 128^3 anisotropic Laplace)"
REF_ARM_TIMEOUT_S = 1700           # the driver's per-step limit is 1800 s
BENCH_BUDGET_S = 1700              # the GPU arm's cpu_baseline gets what is left of this
# PCG iterations of the reference itself per BASELINE config (reference runs:
# tests/golden/cfg1.npz, cfg2.npz, cfg4_full.npz)
REF_ITERS = {1: 12, 2: 16, 3: 64, 4: 49, 5: 36}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler(object):
    """Clocks and throttle reasons during the timed region: one background
    `nvidia-smi --query-gpu=... -lms 200` process (B200_PROFILING.md clocks
    line), started before and stopped after the region.  (Spawning a fresh
    nvidia-smi per sample re-initialises NVML each time and perturbed the
    host-driven PCG loop.)"""

    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self._p = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            for line in self._p.stdout:
                line = line.strip()
                if line:
                    self.rows.append([v.strip() for v in line.split(",")])
        except Exception:
            pass

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                        "--format=csv,noheader,nounits", "-lms", "200"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t.start()
            time.sleep(0.3)  # first sample before the region starts
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
        if self._t.is_alive():
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(backend="nccl", same_gpu=False):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if same_gpu else int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return ws, rank, local


def allmax(v, ws):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def run_reference_subprocess(cfg, threads, timeout_s, n=None):
    """The reference package (oracle/_ref) on one BASELINE config in a child
    process with `threads` BLAS threads (fixed before numpy loads).  Returns
    (result dict or None, error string or None, wall seconds)."""
    env = dict(os.environ)
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        env[k] = str(threads)
    cmd = [sys.executable, os.path.join(ROOT, "oracle", "ref_bench.py"), "--cfg", str(cfg)]
    if n:
        cmd += ["--n", str(n)]
    t = time.perf_counter()
    try:
        p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=max(timeout_s, 1))
    except subprocess.TimeoutExpired:
        return None, f"did not finish within {timeout_s:.0f} s", time.perf_counter() - t
    wall = time.perf_counter() - t
    if p.returncode != 0:
        return None, (p.stderr.strip().splitlines() or ["failed"])[-1][:300], wall
    try:
        return json.loads(p.stdout.strip().splitlines()[-1]), None, wall
    except Exception as e:  # noqa: BLE001
        return None, f"unparsable output: {e}", wall


# ---------------------------------------------------------------------------
def run_reference(args, ws, rank):
    """--impl reference: the reference package itself (oracle/_ref) on the full
    cfg4 problem, one factorize + pcg (reference bench.py:157-166 protocol)
    with every host core as BLAS threads (--ref-threads 1: the single-thread
    figure of BASELINE.md section 2).  One full-size step takes 7-10 minutes
    (measured on the GPU box's 16-core host: 438.7 s with 16 threads, 556.7 s
    with one; profiles/r02_bench_reference_arm.jsonl), so exactly one step is
    run whatever --steps/--warmup say, and the line reports the steps
    actually run."""
    if rank != 0:
        return
    t0 = time.perf_counter()
    threads = args.ref_threads if args.ref_threads > 0 else (os.cpu_count() or 1)
    res, err, wall = run_reference_subprocess(CFG, threads, REF_ARM_TIMEOUT_S)
    base = {"impl": "reference", "metric": METRIC, "unit": "s", "n_gpus": ws, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic"}
    if res is None:
        print(json.dumps({**base, "unavailable": f"reference run failed: {err}"}), flush=True)
        return
    v = res["t_factor_s"] + res["t_solve_s"]
    line = {
        **base, "value": v, "steps": 1, "warmup": 0, "requested_steps": args.steps,
        "requested_warmup": args.warmup, "ms_per_step": v * 1e3,
        "config": {"workload": f"cfg{CFG}-aniso-128" if CFG == 4 else f"cfg{CFG}", "grid": res["grid"],
                   "n": res["n"], "b": res["b"], "rank_tol": res["rank_tol"], "scheme": "nest-2-2", "degree": 1,
                   "pcg_rtol": 1e-12, "parallelism": f"cpu, {threads} BLAS thread(s)"},
        "t_factor_s": res["t_factor_s"], "t_solve_s": res["t_solve_s"], "pcg_iterations": res["iterations"],
        "flops_factorize": res["flops_factorize"], "fp64_tflops_factorize": res["flops_factorize"] / res["t_factor_s"] / 1e12,
        "cpu_baseline": {"value": v, "unit": "s", "cores": threads, "kind": "reference",
                         "sample": f"the whole cfg{CFG} workload (n={res['n']}), one factorize + pcg of the reference "
                                   f"package (oracle/_ref, polyprec {res['polyprec']}), OPENBLAS_NUM_THREADS={threads}, "
                                   f"host {res['cpu_count']} cpus; problem generation {res['t_generate_s']:.1f} s "
                                   f"not timed"},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_wall_s": wall, "arm_wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_sgf(args, ws, rank, local):
    import torch

    import paper_1907_03406_b200 as sgf
    from paper_1907_03406_b200 import _native as N
    from paper_1907_03406_b200 import sharded as S
    from paper_1907_03406_b200.problems import CONFIGS, config_rhs

    torch.cuda.set_device(local)
    c = CONFIGS[CFG]
    prob = c["make"]()
    A = prob.matrix.tocsr()
    A.sort_indices()
    rhs = config_rhs(prob.n, c["seed"])
    opts = dict(scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"], device=local)
    # inputs resident in HBM
    vals = torch.tensor(A.data, dtype=torch.float64, device="cuda")
    ip = torch.tensor(A.indptr, dtype=torch.int64, device="cuda")
    ix = torch.tensor(A.indices, dtype=torch.int32, device="cuda")
    b_dev = torch.tensor(rhs, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    Ad = sgf.DeviceCSR(device=local, indptr=ip, indices=ix, values=vals, n=prob.n)
    ctx = N.context(local)
    stream = torch.cuda.ExternalStream(N.lib().sgf_stream(ctx))

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def step_device(rec=None):
        e0 = ev()
        if ws > 1:
            P = S.factorize_sharded(prob, device_values=vals, **opts)
            e1 = ev()
            x, rep = S.pcg_sharded(A, b_dev, P, tol=1e-12)  # host pattern: halo plan (built once)
        else:
            P = sgf.factorize(prob, device_values=vals, **opts)
            e1 = ev()
            x, rep = sgf.pcg(Ad, b_dev, precond=P, tol=1e-12)
        e2 = ev()
        if rec is not None:
            rec.append((e0, e1, e2, P.stats, rep))
        del P
        return x

    def step_e2e(rec=None):
        e0 = ev()
        if ws > 1:
            P = S.factorize_sharded(prob, **opts)
            x, rep = S.pcg_sharded(A, rhs, P, tol=1e-12)
        else:
            P = sgf.factorize(prob, **opts)
            x, rep = sgf.pcg(A, rhs, precond=P, tol=1e-12)
        e1 = ev()
        if rec is not None:
            rec.append((e0, e1, rep))
        del P
        return x

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    barrier(ws)
    launches0 = N.kernel_launches()
    rec = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t_start = ev()
        for _ in range(args.steps):
            x = step_device(rec)
        t_end = ev()
        torch.cuda.synchronize()
    launches = N.kernel_launches() - launches0
    ms = t_start.elapsed_time(t_end) / args.steps
    ms = allmax(ms, ws)
    tF = float(np.mean([r[0].elapsed_time(r[1]) for r in rec])) / 1e3
    tS = float(np.mean([r[1].elapsed_time(r[2]) for r in rec])) / 1e3
    stats, rep = rec[-1][3], rec[-1][4]
    resid = float(np.linalg.norm(rhs - A @ x.cpu().numpy()) / np.linalg.norm(rhs))

    # end to end through the public API with host buffers
    for _ in range(1):
        step_e2e()
    torch.cuda.synchronize()
    barrier(ws)
    rec2 = []
    for _ in range(args.steps):
        step_e2e(rec2)
    torch.cuda.synchronize()
    e2e_ms = allmax(float(np.mean([r[0].elapsed_time(r[1]) for r in rec2])), ws)
    h2d = 8 * A.nnz + 8 * prob.n * stats_pi(stats) + (8 * (prob.n + 1) + 4 * A.nnz + 8 * A.nnz) + 8 * prob.n
    d2h = 8 * prob.n

    # roofline of the dominant kernel class from one instrumented step
    N.profile_enable(True)
    if ws > 1:
        step_device()
        sparse = None
    else:
        Pp = sgf.factorize(prob, device_values=vals, **opts)
        sgf.pcg(Ad, b_dev, precond=Pp, tol=1e-12)
    torch.cuda.synchronize()
    prof = N.profile_read()
    N.profile_enable(False)
    if ws == 1:
        # the apply streams only the couplings' 32-column tiles that hold a
        # nonzero (apply.cpp); the profiler's work is the dense formula
        # (SURVEY 8d).  Per apply: 2 sweeps over the couplings.
        N.profile_enable(True)
        Pp.apply_inverse(b_dev)
        torch.cuda.synchronize()
        p1 = N.profile_read()
        N.profile_enable(False)
        ed, enz = coupling_bytes(Pp)
        n_app = prof["gemv"][2] / max(p1["gemv"][2], 1)
        sparse = {"applies": n_app, "coupling_bytes_dense_per_sweep": ed, "coupling_bytes_nonzero_per_sweep": enz,
                  "gemv_bytes_dense": prof["gemv"][1], "gemv_bytes_nonzero": prof["gemv"][1] - n_app * 2 * (ed - enz)}
        del Pp
    pk, pk_kind = peaks()
    dom = max(prof, key=lambda k: prof[k][0])
    mss, work, nl = prof[dom]
    if dom == "gemv" and sparse:
        work = sparse["gemv_bytes_nonzero"]
    if dom == "gemm_int8emu":
        # FP64 products on the INT8 tensor cores: 36 int8 slice products per
        # FP64 product (ozaki.cu); achieved/peak in INT8 tensor ops
        achieved = 36.0 * work / (mss * 1e-3) / 1e12
        roof = {"bound": "tensor", "pipe": "tcgen05 kind::i8 (FP64 emulated, 8 slices)", "achieved": achieved,
                "peak": INT8_PEAK_TOPS, "unit": "TOPS", "frac": achieved / INT8_PEAK_TOPS,
                "fp64_equivalent_tflops": work / (mss * 1e-3) / 1e12, "peak_source": INT8_PEAK_SOURCE}
    elif dom == "gemm":
        achieved = work / (mss * 1e-3) / 1e12
        roof = {"bound": "tensor", "pipe": "DMMA (FP64 mma.sync; tcgen05 has no f64 kind)", "achieved": achieved,
                "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS,
                "peak_source": "measured DMMA f64 issue rate (tools/fp64_peak.cu, profiles/fp64_peak_r01.jsonl); "
                               "MEASURED_PEAKS.json has no FP64 figure"}
    else:
        achieved = work / (mss * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "peak_source": pk_kind}
        if dom == "gemv" and sparse:
            roof["algorithmic_bytes"] = ("the factor entries the sweeps must read: triangles, compression blocks "
                                         "and the couplings' 32-column tiles that hold a nonzero (all-zero tiles "
                                         "of the block-sparse couplings are skipped)")
            roof["dense_equivalent_gbs"] = sparse["gemv_bytes_dense"] / (mss * 1e-3) / 1e9
            roof["sparsity"] = sparse
    roof.update({"kernel": dom, "launches": int(nl), "ms_per_step": mss, "traffic": traffic_from_profiles(dom),
                 "classes_ms": {k: round(v[0], 3) for k, v in prof.items()}})
    gemv = prof["gemv"]
    spmv = prof["spmv"]
    extra = {} if rank != 0 else {
        "fp64_tflops_factorize": stats["flops_factorize"] / tF / 1e12,
        "t_factor_s": tF, "t_solve_s": tS, "pcg_iterations": rep.iterations,
        "reference_pcg_iterations": 49, "final_rel_residual": rep.final_rel_residual, "check_residual": resid,
        "gemm_tflops": prof["gemm"][1] / max(prof["gemm"][0], 1e-9) / 1e9,
        "int8emu_fp64_tflops": prof["gemm_int8emu"][1] / max(prof["gemm_int8emu"][0], 1e-9) / 1e9,
        "int8emu_ms": prof["gemm_int8emu"][0], "int8emu_split_ms": prof["int8emu_split"][0],
        "apply_gemv_gbs": (sparse["gemv_bytes_nonzero"] if sparse else gemv[1]) / max(gemv[0], 1e-9) / 1e6,
        "spmv_gbs": spmv[1] / max(spmv[0], 1e-9) / 1e6,
        "note_dense_equivalent": "fp64_tflops_factorize and int8emu_fp64_tflops divide the reference's dense flop "
                                 "tally; the emulated products skip K tiles where an operand tile is all zero "
                                 "(block-sparse couplings), so these are dense-equivalent rates",
    }

    # the same headline step with every FP64 product on IEEE DMMA (no INT8
    # emulation): what the factorization costs in native FP64
    ieee = None
    if ws == 1 and not args.no_extras:
        os.environ["SGF_OZAKI_MIN_M"] = "0"
        try:
            step_device()
            torch.cuda.synchronize()
            rec3 = []
            for _ in range(max(1, min(args.steps, 3))):
                step_device(rec3)
            torch.cuda.synchronize()
        finally:
            del os.environ["SGF_OZAKI_MIN_M"]
        tFi = float(np.mean([r[0].elapsed_time(r[1]) for r in rec3])) / 1e3
        tSi = float(np.mean([r[1].elapsed_time(r[2]) for r in rec3])) / 1e3
        ieee = {"value": tFi + tSi, "unit": "s", "steps": len(rec3), "t_factor_s": tFi, "t_solve_s": tSi,
                "pcg_iterations": rec3[-1][4].iterations,
                "executed_fp64_tflops": rec3[-1][3]["flops_factorize"] / tFi / 1e12,
                "fp64_peak_tflops": FP64_PEAK_TFLOPS,
                "note": "SGF_OZAKI_MIN_M=0: every dense FP64 product on DMMA (IEEE FP64); the reference flop "
                        "tally / t_F; level-1 sparse gathers count as their reference flops"}
    del Ad

    # every BASELINE config: factor / apply / solve (device-resident inputs)
    configs = {}
    if ws == 1 and not args.no_extras:
        for k in (1, 2, 3, 4, 5):
            configs[f"cfg{k}"] = measure_config(k, local)

    cpu = None
    if rank == 0 and ws == 1 and args.cpu_baseline != "none":
        left = BENCH_BUDGET_S - (time.perf_counter() - T_START)
        threads = os.cpu_count() or 1
        n_sample = None if args.cpu_baseline == "full" else 40
        res, err, wall = run_reference_subprocess(CFG, threads, left, n=n_sample)
        if res is not None:
            cpu = {"value": res["t_factor_s"] + res["t_solve_s"], "unit": "s", "cores": threads, "kind": "reference",
                   "t_factor_s": res["t_factor_s"], "t_solve_s": res["t_solve_s"], "pcg_iterations": res["iterations"],
                   "sample": (f"the whole cfg{CFG} workload (n={res['n']}): one factorize + pcg of the reference "
                              f"package (oracle/_ref, polyprec {res['polyprec']}), OPENBLAS_NUM_THREADS={threads} "
                              f"(all host cores), timed as reference bench.py:157-166"
                              if n_sample is None else
                              f"bounded sample: the cfg{CFG} operator on a {n_sample}^3 grid (n={res['n']}), "
                              f"reference package, OPENBLAS_NUM_THREADS={threads}; not the bench config")}
        else:
            cpu = {"value": None, "unit": "s", "cores": threads, "kind": "reference",
                   "sample": f"reference run on the whole cfg{CFG} workload with {threads} BLAS threads: {err}"}
    if rank == 0:
        line = {
            "metric": "factor+solve wall time (cfg4: 128^3 anisotropic Laplace)", "value": ms / 1e3, "unit": "s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "cfg4-aniso-128" if CFG == 4 else f"cfg{CFG}-code-path-check-not-a-bench-value",
                       "grid": list(prob.grid.dims), "n": prob.n, "nnz": int(A.nnz),
                       "b": c["b"], "rank_tol": c["rank_tol"], "scheme": "nest-2-2", "degree": 1,
                       "pcg_rtol": 1e-12, "parallelism": f"shard{ws}" if ws > 1 else "single",
                       "l2": "inputs and factors (>60 GB) exceed the 126 MB L2",
                       "fp64_products": "DMMA (mma.sync f64) for nodes < 640 unknowns; FP64 emulated on the "
                                        "tcgen05 INT8 tensor cores (Ozaki scheme, 8 balanced 8-bit digits, 62-bit, exact "
                                        "int32 accumulation; all-zero operand tiles skipped) for larger nodes"},
            "e2e": {"value": e2e_ms / 1e3, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches), "clocks": clk.summary(), "roofline": roof, "cpu_baseline": cpu,
            "ieee_fp64": ieee, "configs": configs,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)


def measure_config(k, local, steps=2):
    """t_F, t_S, iterations, apply time / bandwidth and FP64 rate for BASELINE
    config k with device-resident CSR values and RHS (one warm-up step)."""
    import torch

    import paper_1907_03406_b200 as sgf
    from paper_1907_03406_b200 import _native as N
    from paper_1907_03406_b200.problems import CONFIGS, config_rhs

    c = CONFIGS[k]
    prob = c["make"]()
    A = prob.matrix.tocsr()
    A.sort_indices()
    rhs = config_rhs(prob.n, c["seed"])
    opts = dict(scheme="nest-2-2", degree=1, b=c["b"], rank_tol=c["rank_tol"], device=local)
    vals = torch.tensor(A.data, dtype=torch.float64, device="cuda")
    Ad = sgf.DeviceCSR(device=local, indptr=torch.tensor(A.indptr, dtype=torch.int64, device="cuda"),
                       indices=torch.tensor(A.indices, dtype=torch.int32, device="cuda"), values=vals, n=prob.n)
    b_dev = torch.tensor(rhs, dtype=torch.float64, device="cuda")
    stream = torch.cuda.ExternalStream(N.lib().sgf_stream(N.context(local)))

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    out = []
    for s in range(steps + 1):
        e0 = ev()
        P = sgf.factorize(prob, device_values=vals, **opts)
        e1 = ev()
        x, rep = sgf.pcg(Ad, b_dev, precond=P, tol=1e-12)
        e2 = ev()
        torch.cuda.synchronize()
        if s:
            out.append((e0.elapsed_time(e1) / 1e3, e1.elapsed_time(e2) / 1e3, rep))
        if s < steps:
            del P
    # apply_inverse alone: time and the bytes its sweeps stream (native profile)
    y = torch.empty_like(b_dev)
    for _ in range(2):
        y = P.apply_inverse(b_dev)
    torch.cuda.synchronize()
    N.profile_enable(True)
    a0 = ev()
    na = 5
    for _ in range(na):
        y = P.apply_inverse(b_dev)
    a1 = ev()
    torch.cuda.synchronize()
    prof = N.profile_read()
    N.profile_enable(False)
    ms_apply = a0.elapsed_time(a1) / na
    apply_bytes = sum(prof[c][1] for c in ("gemv", "copy", "vec")) / na
    ed, enz = coupling_bytes(P)
    apply_bytes_nz = apply_bytes - 2 * (ed - enz)
    tF = float(np.mean([o[0] for o in out]))
    tS = float(np.mean([o[1] for o in out]))
    rep = out[-1][2]
    st = P.stats
    return {"grid": list(prob.grid.dims), "n": prob.n, "nnz": int(A.nnz), "b": c["b"], "rank_tol": c["rank_tol"],
            "t_factor_s": tF, "t_solve_s": tS, "factor_plus_solve_s": tF + tS, "steps": steps,
            "pcg_iterations": rep.iterations, "reference_pcg_iterations": REF_ITERS[k],
            "final_rel_residual": rep.final_rel_residual,
            "fp64_tflops_factorize": st["flops_factorize"] / tF / 1e12,
            "fp64_frac_of_dmma_peak": st["flops_factorize"] / tF / 1e12 / FP64_PEAK_TFLOPS,
            "ms_per_apply": ms_apply, "apply_gbs": apply_bytes_nz / (ms_apply * 1e-3) / 1e9,
            "apply_frac_of_hbm": apply_bytes_nz / (ms_apply * 1e-3) / 1e9 / peaks()[0]["hbm_gbs"],
            "apply_gb": apply_bytes_nz / 1e9, "apply_gb_dense": apply_bytes / 1e9,
            "flops_factorize": st["flops_factorize"], "flops_apply": st["flops_apply"]}


def coupling_bytes(P):
    """(dense, nonzero-tile) bytes of the preconditioner's couplings per sweep."""
    from paper_1907_03406_b200 import _native as N

    out = np.zeros(2)
    N.raise_for(N.lib().sgf_precond_coupling_bytes(P._h, out.ctypes.data), P._ctx)
    return float(out[0]), float(out[1])


def stats_pi(stats):
    return 4  # degree-1 scalar basis columns


def traffic_from_profiles(kernel):
    """dram bytes per launch of the dominant kernel from a committed ncu
    capture summary (profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


T_START = time.perf_counter()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sgf", choices=["sgf", "reference"])
    ap.add_argument("--cpu-baseline", default="sample", choices=["full", "sample", "none"],
                    help="GPU arm's CPU reference leg: a bounded sample, the reference package on the cfg4 "
                         "operator at 40^3 with all host cores (default, ~15-20 s); the whole cfg4 run on all "
                         "host cores (~15 min; profiles/r02_bench_cpu_full.jsonl); or none.  The full-size "
                         "single-thread reference is the --impl reference arm")
    ap.add_argument("--no-extras", action="store_true", help="skip the per-config and IEEE-FP64 lines")
    ap.add_argument("--ref-threads", type=int, default=0,
                    help="--impl reference: BLAS threads of the reference run (0: every host core; 1: single thread)")
    # code-path checks only (numbers from these are not bench values): another
    # config, gloo collectives, every rank on GPU 0
    ap.add_argument("--cfg", type=int, default=4)
    ap.add_argument("--dist-backend", default="nccl")
    ap.add_argument("--same-gpu", action="store_true")
    args = ap.parse_args()
    global CFG
    CFG = args.cfg
    ws, rank, local = dist_setup(args.dist_backend, args.same_gpu) if args.impl == "sgf" else (int(os.environ.get("WORLD_SIZE", "1")),
                                                             int(os.environ.get("RANK", "0")), 0)
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_sgf(args, ws, rank, local)
    if ws > 1 and args.impl == "sgf":
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
