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

Run:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sgf|reference]
N > 1 (torchrun, NCCL): the one 128^3 problem is sharded across the ranks
(sharded.py: subtree ownership of the nested-dissection tree, rank-local
elimination phase, trailing-matrix reduction onto rank 0, collective apply
inside PCG); strong scaling, the step time is the max over ranks.
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
SURVEY_REF_FULL_S = 682.4 + 270.4  # reference at full cfg4 size, 1 BLAS thread
CPU_SAMPLE_N = 40                  # bounded CPU sample: the same operator on a 40^3 grid


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


def cpu_reference_step(sample_n):
    """One bounded CPU step of the reference algorithm (oracle port): factorize
    + pcg on the cfg4 operator at sample_n^3.  Returns (t_F, t_S, stats, iters)."""
    from oracle import sgf_oracle as O
    from paper_1907_03406_b200 import problems as pr

    c = pr.CONFIGS[CFG]
    p = pr.anisotropic7(sample_n, 1e-3)
    rhs = pr.config_rhs(p.n, c["seed"])
    t = time.perf_counter()
    P = O.factorize(p.matrix, p.coords, p.grid.dims, 1, scheme="nest-2-2", degree=1, b=c["b"],
                    rank_tol=c["rank_tol"])
    tf = time.perf_counter() - t
    t = time.perf_counter()
    x, rep = O.pcg(p.matrix, rhs, P.apply_inverse, tol=1e-12)
    ts = time.perf_counter() - t
    return tf, ts, P.stats, rep.iterations


def extrapolate(tf, ts, st, it, full):
    """Scale a sample's times to the full config: factorization by the
    reference flop tally, solve by apply work x (iterations + 1)."""
    ef = tf * full["flops_factorize"] / st["flops_factorize"]
    es = ts * (full["flops_apply"] * (full["iters"] + 1)) / (st["flops_apply"] * (it + 1))
    return ef, es


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
def run_reference(args, ws, rank):
    """--impl reference: the reference's CPU algorithm (oracle port; the
    Python reference itself is not present on the GPU box) on bounded samples
    of the workload, reported in the same unit as the GPU arm."""
    if rank != 0:
        return
    full = {"flops_factorize": 11816662185330, "flops_apply": 14116631728, "iters": 49}  # cfg4
    times = []
    for s in range(args.warmup + args.steps):
        tf, ts, st, it = cpu_reference_step(CPU_SAMPLE_N)
        if s >= args.warmup:
            times.append(extrapolate(tf, ts, st, it, full) + (tf, ts))
    ef = float(np.mean([t[0] for t in times]))
    es = float(np.mean([t[1] for t in times]))
    v = ef + es
    sample = (f"anisotropic 7-point diag(1,1,1e-3) on {CPU_SAMPLE_N}^3 (n={CPU_SAMPLE_N ** 3}), "
              f"nest-2-2 b=9 rank_tol 1e-3: t_F {np.mean([t[2] for t in times]):.2f}s, "
              f"t_S {np.mean([t[3] for t in times]):.2f}s, scaled to 128^3 by reference flops_factorize "
              f"and flops_apply x (iterations+1)")
    line = {
        "impl": "reference", "metric": "factor+solve wall time (cfg4: 128^3 anisotropic Laplace)",
        "value": v, "unit": "s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": {"workload": "cfg4-aniso-128", "grid": [128, 128, 128],
                                                         "n": 2097152, "b": 9, "rank_tol": 1e-3, "pcg_rtol": 1e-12},
        "t_factor_s": ef, "t_solve_s": es,
        "cpu_baseline": {"value": v, "unit": "s", "cores": blas_threads(), "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "survey_reference_full_s": SURVEY_REF_FULL_S,
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
            x, rep = S.pcg_sharded(Ad, b_dev, P, tol=1e-12)
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
    step_device()
    torch.cuda.synchronize()
    prof = N.profile_read()
    N.profile_enable(False)
    pk, pk_kind = peaks()
    dom = max(prof, key=lambda k: prof[k][0])
    mss, work, nl = prof[dom]
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
        "apply_gemv_gbs": gemv[1] / max(gemv[0], 1e-9) / 1e6, "spmv_gbs": spmv[1] / max(spmv[0], 1e-9) / 1e6,
    }

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        full = {"flops_factorize": stats["flops_factorize"], "flops_apply": stats["flops_apply"],
                "iters": rep.iterations}
        tf, ts, st, it = cpu_reference_step(CPU_SAMPLE_N)
        ef, es = extrapolate(tf, ts, st, it, full)
        cpu = {"value": ef + es, "unit": "s", "cores": blas_threads(), "kind": "port",
               "sample": f"oracle (numpy port of the reference) on the cfg4 operator at {CPU_SAMPLE_N}^3: "
                         f"t_F {tf:.2f}s + t_S {ts:.2f}s ({it} iterations), scaled to 128^3 by flops_factorize "
                         f"and flops_apply x (iterations+1); reference measured at full size in SURVEY: "
                         f"{SURVEY_REF_FULL_S:.0f}s"}
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
                       "fp64_products": "DMMA (mma.sync f64) for nodes < 1024 unknowns; FP64 emulated on the "
                                        "tcgen05 INT8 tensor cores (Ozaki scheme, 8 x 7-bit slices, 56-bit, exact "
                                        "int32 accumulation) for larger nodes"},
            "e2e": {"value": e2e_ms / 1e3, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches), "clocks": clk.summary(), "roofline": roof, "cpu_baseline": cpu,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sgf", choices=["sgf", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
