"""ctypes binding of the C ABI in include/sgf.h (libsgf.so, built in-tree).

There is no CPU fallback: importing the package works without a GPU (so the
host-side logic can be tested), but every compute entry point goes through
`lib()` / `context()`, which raise `NativeUnavailable` when the shared
library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
# SGF_LIB: alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("SGF_LIB") or os.path.join(_HERE, "libsgf.so")

SGF_OK, SGF_NOT_SPD, SGF_SHAPE, SGF_INDEFINITE, SGF_INVALID_ARG, SGF_TRACE, SGF_CUDA, SGF_OOM, SGF_NON_SYMMETRIC = range(9)
MODE = {"polynomial": 0, "lowrank": 1, "exact": 2}
APPLY_INVERSE, APPLY_HALF_INVERSE, APPLY_HALF_INVERSE_T, APPLY_OPERATOR = range(4)
FACTOR_TYPES = {0: "EliminationFactor", 1: "CompressionFactor", 2: "DenseFactor"}
SOLVE_FORWARD, SOLVE_TRANSPOSE, MULT_TRANSPOSE, MULT_FORWARD = range(4)

# functions the header declares (checked by tests/test_native_abi.py)
EXPORTS = (
    "sgf_create", "sgf_destroy", "sgf_last_error", "sgf_stream", "sgf_sync", "sgf_trim", "sgf_factorize",
    "sgf_precond_free", "sgf_precond_n", "sgf_precond_stats_json", "sgf_precond_rank_trace",
    "sgf_precond_num_factors", "sgf_precond_coupling_bytes", "sgf_precond_coupling_bytes_level", "sgf_precond_coupling_bytes_detail", "sgf_precond_factor_info", "sgf_precond_factor_copy", "sgf_apply",
    "sgf_csr_create", "sgf_csr_free", "sgf_spmv", "sgf_pcg", "sgf_pcg_cb",
    "sgf_precond_shard_info", "sgf_precond_shard_set", "sgf_apply_part", "sgf_cell_unknowns",
    "sgf_kernel_launches", "sgf_profile_enable", "sgf_profile_read", "sgf_pcg_ops", "sgf_memcpy",
    "sgf_stream_wait", "sgf_factor_apply", "sgf_potrf_batched", "sgf_trsm_batched", "sgf_qrcp_batched", "sgf_gemm",
    "sgf_exchange_accumulate", "sgf_apply_shard", "sgf_vec_gather", "sgf_vec_scatter", "sgf_pcg_dist",
)
PROF_CLASSES = ("gemm", "gemv", "spmv", "qr", "chol", "copy", "vec", "gemm_int8emu", "int8emu_split")


class NativeUnavailable(RuntimeError):
    """The CUDA implementation cannot run here (library or GPU missing)."""


class FactorArgs(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("nnz", C.c_int64),
        ("indptr", C.c_void_p), ("indices", C.c_void_p), ("values", C.c_void_p),
        ("values_on_device", C.c_int),
        ("pi_cols", C.c_int), ("phi", C.c_void_p),
        ("nlevels", C.c_int), ("level_ncells", C.c_void_p), ("cell_kind", C.c_void_p),
        ("cell_interior", C.c_void_p), ("father", C.c_void_p),
        ("l1_ptr", C.c_void_p), ("l1_unknowns", C.c_void_p),
        ("compress_kind_mask", C.c_int), ("raw_kind_mask", C.c_int), ("skip_levels", C.c_int),
        ("compression", C.c_int), ("mode", C.c_int), ("rank_tol", C.c_double),
        ("n_trace", C.c_int), ("trace", C.c_void_p),
        ("n_replay", C.c_int), ("replay_ptr", C.c_void_p), ("replay_perm", C.c_void_p),
        ("coords", C.c_void_p), ("n_vertices", C.c_int64), ("degree", C.c_int), ("components", C.c_int),
        ("shard_rank", C.c_int), ("shard_count", C.c_int), ("cell_rank", C.c_void_p),
        ("shard_stop_level", C.c_int), ("exchange", C.c_void_p), ("exchange_user", C.c_void_p),
    ]


class Exchange(C.Structure):
    """sgf_exchange (include/sgf.h): one rank's trailing-matrix contribution."""
    _fields_ = [("nblocks", C.c_int64), ("nsend", C.c_int64), ("send_idx", C.POINTER(C.c_int32)),
                ("send_meta", C.POINTER(C.c_int32)), ("send_buf", C.c_void_p), ("send_len", C.c_int64),
                ("accum", C.c_void_p)]


# int exchange(void* user, const sgf_exchange* x)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(Exchange))
# int reduce(void* user, double* vals, int n)
REDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int)
# int precond(void* user, const double* in, double* out)
PRECOND_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)
# int matvec(void* user, const double* in, double* out)
MATVEC_FN = PRECOND_FN


class PcgReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("final_rel_residual", C.c_double),
                ("wall_time", C.c_double), ("history_len", C.c_int)]


_lib = None
_lock = threading.Lock()
_ctx = {}
_ctx_device = {}


def load_library(path=LIB_PATH):
    """Load libsgf.so and declare signatures (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(path)
        vp, i32, i64, d = C.c_void_p, C.c_int, C.c_int64, C.c_double
        sig = {
            "sgf_create": (i32, [C.POINTER(vp), i32]),
            "sgf_destroy": (i32, [vp]),
            "sgf_last_error": (C.c_char_p, [vp]),
            "sgf_stream": (vp, [vp]),
            "sgf_sync": (i32, [vp]),
            "sgf_trim": (i32, [vp]),
            "sgf_factorize": (i32, [vp, C.POINTER(FactorArgs), C.POINTER(vp)]),
            "sgf_precond_free": (i32, [vp]),
            "sgf_precond_n": (i64, [vp]),
            "sgf_precond_stats_json": (C.c_char_p, [vp]),
            "sgf_precond_rank_trace": (i32, [vp, vp, i32]),
            "sgf_precond_num_factors": (i32, [vp]),
            "sgf_precond_coupling_bytes": (i32, [vp, vp]),
            "sgf_precond_coupling_bytes_level": (i32, [vp, i32, vp]),
            "sgf_precond_coupling_bytes_detail": (i32, [vp, i32, vp]),
            "sgf_precond_factor_info": (i32, [vp, i32, vp]),
            "sgf_precond_factor_copy": (i32, [vp, i32, i32, vp, i64]),
            "sgf_apply": (i32, [vp, i32, vp, vp, i32]),
            "sgf_csr_create": (i32, [vp, i64, i64, vp, vp, vp, i32, C.POINTER(vp)]),
            "sgf_csr_free": (i32, [vp]),
            "sgf_spmv": (i32, [vp, vp, vp, i32]),
            "sgf_pcg": (i32, [vp, vp, vp, vp, vp, d, i32, i32, i32, C.POINTER(PcgReport), vp]),
            "sgf_pcg_cb": (i32, [vp, vp, PRECOND_FN, vp, vp, vp, d, i32, i32, i32, C.POINTER(PcgReport), vp]),
            "sgf_precond_shard_info": (i32, [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
            "sgf_precond_shard_set": (i32, [vp, i32, vp, i64]),
            "sgf_apply_part": (i32, [vp, i32, vp]),
            "sgf_cell_unknowns": (i32, [i32, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, i32, vp, vp]),
            "sgf_pcg_ops": (i32, [vp, i64, vp, MATVEC_FN, vp, vp, PRECOND_FN, vp, vp, vp, d, i32, i32, i32,
                                  C.POINTER(PcgReport), vp]),
            "sgf_memcpy": (i32, [vp, vp, vp, i64]),
            "sgf_stream_wait": (i32, [vp, vp]),
            "sgf_factor_apply": (i32, [vp, i32, i32, vp, i32]),
            "sgf_potrf_batched": (i32, [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp]),
            "sgf_trsm_batched": (i32, [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
            "sgf_qrcp_batched": (i32, [vp, i32, vp, vp, vp, vp, d, i32, vp, vp, vp, vp, vp]),
            "sgf_gemm": (i32, [vp, i32, i32, i32, d, vp, i32, vp, i32, d, vp, i32]),
            "sgf_exchange_accumulate": (i32, [vp, vp, i64, vp]),
            "sgf_apply_shard": (i32, [vp, i32, vp, vp, vp, i32]),
            "sgf_vec_gather": (i32, [vp, vp, vp, vp, i64]),
            "sgf_vec_scatter": (i32, [vp, vp, vp, vp, i64]),
            "sgf_pcg_dist": (i32, [vp, i64, MATVEC_FN, vp, PRECOND_FN, vp, REDUCE_FN, vp, vp, vp, d, i32, i32,
                                   C.POINTER(PcgReport), vp]),
            "sgf_kernel_launches": (C.c_uint64, []),
            "sgf_profile_enable": (i32, [i32]),
            "sgf_profile_read": (i32, [vp, i32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def lib():
    return load_library()


def raise_for(status, ctx=None, what=""):
    if status == SGF_OK:
        return
    msg = lib().sgf_last_error(ctx).decode("utf-8", "replace") if ctx is not None else ""
    if what:
        msg = f"{what}: {msg}" if msg else what
    cls = {
        SGF_NOT_SPD: E.NotSPDError,
        SGF_SHAPE: E.ShapeMismatchError,
        SGF_INDEFINITE: E.IndefiniteDetectedError,
        SGF_INVALID_ARG: ValueError,
        SGF_TRACE: RuntimeError,
        SGF_NON_SYMMETRIC: E.NonSymmetricPatternError,
        SGF_OOM: MemoryError,
    }.get(status, E.DeviceError)
    raise cls(msg)


def context(device=0):
    """The per-device native context (created on first use)."""
    with _lock:
        if device in _ctx:
            return _ctx[device]
    L = lib()
    h = C.c_void_p()
    st = L.sgf_create(C.byref(h), int(device))
    if st != SGF_OK:
        msg = L.sgf_last_error(None).decode()
        raise NativeUnavailable(f"cannot create a CUDA context on device {device}: {msg}")
    with _lock:
        _ctx[device] = h
        _ctx_device[h.value] = int(device)
    return h


def trim_memory():
    """Return the device memory the library caches for reuse (on every device
    with a context) to the driver; live factors and matrices are untouched.
    For a process that shares its GPU with others, e.g. a test session about
    to launch worker processes on the same device."""
    with _lock:
        handles = list(_ctx.values())
    for h in handles:
        raise_for(lib().sgf_trim(h), h)


def context_device(ctx):
    """The CUDA device index a native context was created on."""
    return _ctx_device[ctx.value]


def order_after_torch(ctx, device=None):
    """Make the native context stream wait for everything enqueued so far on
    torch's current stream of the context's device: a tensor a torch kernel
    is still producing is not read early (the native stream is a separate,
    non-blocking stream).  Native calls synchronise their own stream before
    returning, so their outputs are ready for torch."""
    import torch

    dev = context_device(ctx) if device is None else device
    s = torch.cuda.current_stream(dev).cuda_stream
    raise_for(lib().sgf_stream_wait(ctx, C.c_void_p(s)), ctx)


def check_device_tensor(t, dtype, device, what):
    """Validate a CUDA tensor handed to the native code by pointer: dtype,
    contiguity and device (a mismatch would read out of bounds or garbage)."""
    import torch

    if not getattr(t, "is_cuda", False):
        raise ValueError(f"{what} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{what} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    if t.device.index != device:
        raise ValueError(f"{what} is on cuda:{t.device.index} but the context is on cuda:{device}")
    return torch


def kernel_launches():
    return int(lib().sgf_kernel_launches())


def profile_enable(on=True):
    lib().sgf_profile_enable(1 if on else 0)


def profile_read():
    """{class: (ms, work, launches)} accumulated since profile_enable()."""
    out = np.zeros(3 * len(PROF_CLASSES))
    st = lib().sgf_profile_read(out.ctypes.data, len(out))
    raise_for(st, None)
    return {c: tuple(out[3 * i:3 * i + 3]) for i, c in enumerate(PROF_CLASSES)}


def ptr(a):
    """Data pointer of a contiguous numpy array or a torch tensor."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"], "array must be contiguous"
        return a.ctypes.data
    return a.data_ptr()
