"""ctypes binding of the sm_100a C-ABI library (include/msgpu.h).

The product path has no CPU fallback: if ``libmsgpu.so`` is missing or no
CUDA device is usable, every solver entry point raises.
"""

from __future__ import annotations

import atexit
import ctypes as C
import os
from pathlib import Path

import numpy as np

# MSGPU_LIB: load an alternative build of the same library (kernel-variant sweeps)
LIB_PATH = Path(os.environ.get("MSGPU_LIB") or Path(__file__).resolve().parent / "libmsgpu.so")

MS_OK, MS_E_INVALID, MS_E_NOT_SPD, MS_E_CUDA, MS_E_NOMEM, MS_E_STATE = 0, -1, -2, -3, -4, -5
MS_LEVEL1_NEIGHBORHOODS, MS_LEVEL1_BLOCKS = 0, 1
MS_LOCAL_BANDED, MS_LOCAL_DENSE_INV = 0, 1
MS_L1_ELASTICITY, MS_L1_HEAT = 0, 1
MS_EIG_HEAT, MS_EIG_ELASTICITY = 0, 1
MS_COARSE_INVERSE, MS_COARSE_CHOLESKY = 0, 1

# every symbol include/msgpu.h declares
EXPORTS = (
    "ms_abi_version", "ms_last_error", "ms_ctx_create", "ms_ctx_destroy",
    "ms_problem_create", "ms_problem_destroy", "ms_problem_n_free", "ms_problem_set_modulus",
    "ms_operator_apply", "ms_precond_build", "ms_precond_destroy", "ms_precond_apply",
    "ms_precond_apply_coarse", "ms_precond_info_get", "ms_precond_coarse_matrix", "ms_pcg_solve",
    "ms_ctx_set_profiling", "ms_ctx_profile_get", "ms_ctx_stream", "ms_precond_bench",
    "ms_nccl_unique_id", "ms_ctx_attach_nccl", "ms_ctx_attach_callbacks", "ms_comm_selftest", "ms_strip_rows", "ms_copy", "ms_cache_trim",
    "ms_halo_plan", "ms_ctx_set_profiling_mask", "ms_filter_create", "ms_filter_destroy", "ms_filter_apply", "ms_filter_adjoint",
    "ms_problem_set_density", "ms_compliance_sensitivity", "ms_oc_update", "ms_dot", "ms_unit_element", "ms_dense_spd_solve",
    "ms_csr_create", "ms_csr_apply", "ms_csr_destroy", "ms_pcg_solve_generic",
)

ALLREDUCE_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64)
BROADCAST_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int)
SENDRECV_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_int)


APPLY_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64)
MS_LINOP_NONE, MS_LINOP_PROBLEM, MS_LINOP_PRECOND, MS_LINOP_CSR, MS_LINOP_CALLBACK = range(5)


class LinOp(C.Structure):
    """ms_linop: one operand of ms_pcg_solve_generic."""
    _fields_ = [("kind", C.c_int), ("handle", C.c_void_p), ("fn", APPLY_CB), ("user", C.c_void_p)]


class CommCallbacks(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allreduce_sum", ALLREDUCE_CB), ("broadcast", BROADCAST_CB),
                ("sendrecv", SENDRECV_CB)]
BENCH_NAMES = ("matvec", "level1", "restrict", "coarse_solve", "combine", "combine_l1", "combine_coarse")
PROF_NAMES = ("matvec", "update", "level1", "restrict", "coarse_solve", "combine")
MS_PROF_N = 8


class PrecondOpts(C.Structure):
    _fields_ = [
        ("Nx", C.c_int), ("Ny", C.c_int), ("level1_kind", C.c_int), ("delta", C.c_int),
        ("n_max", C.c_int), ("gap_threshold", C.c_double), ("enrich", C.c_int),
        ("fixed_rule", C.c_int), ("local_solver", C.c_int), ("use_coarse", C.c_int),
        ("heat_dirichlet_nodes", C.POINTER(C.c_int64)), ("n_heat_dirichlet", C.c_int64),
        ("randomized", C.c_int), ("n_snapshots", C.c_int), ("snapshots", C.c_void_p),
        ("level1_operator", C.c_int), ("eig_kind", C.c_int), ("coarse_solve", C.c_int),
    ]


class PrecondInfo(C.Structure):
    _fields_ = [
        ("coarse_dim", C.c_int), ("n_centers", C.c_int), ("n_subdomains", C.c_int),
        ("max_eig_passes", C.c_int), ("mean_eig_passes", C.c_double), ("t_level1", C.c_double), ("t_eig", C.c_double),
        ("t_coarse", C.c_double), ("local_bytes", C.c_double), ("coarse_bytes", C.c_double),
        ("level1_twisted", C.c_int), ("level1_copies", C.c_int), ("n_subdomains_local", C.c_int),
        ("level1_unit", C.c_int),
    ]


class Report(C.Structure):
    _fields_ = [
        ("kernel_launches", C.c_int64), ("iterations", C.c_int), ("converged", C.c_int), ("final_residual", C.c_double),
        ("t_solve", C.c_double), ("t_total", C.c_double),
    ]


class MsError(RuntimeError):
    pass


_lib = None
_SHUTDOWN = False


def _mark_shutdown():
    global _SHUTDOWN
    _SHUTDOWN = True


atexit.register(_mark_shutdown)


def alive():
    """False once the interpreter is exiting: handles are leaked, not freed."""
    return _lib is not None and not _SHUTDOWN


def load(path: str | os.PathLike | None = None):
    """Load and prototype the library (no CUDA call is made here)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} not built: run `make` or __graft_entry__.build() (no CPU fallback)")
    lib = C.CDLL(str(p))
    vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)
    i64p = C.POINTER(C.c_int64)
    sig = {
        "ms_abi_version": (C.c_int, []),
        "ms_last_error": (C.c_int, [vp, C.c_char_p, C.c_size_t]),
        "ms_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "ms_ctx_destroy": (C.c_int, [vp]),
        "ms_problem_create": (C.c_int, [vp, C.c_int, C.c_int, C.c_double, C.c_double, vp, vp,
                                        C.c_int64, C.POINTER(vp)]),
        "ms_problem_destroy": (C.c_int, [vp]),
        "ms_problem_n_free": (C.c_int64, [vp]),
        "ms_problem_set_modulus": (C.c_int, [vp, vp]),
        "ms_operator_apply": (C.c_int, [vp, vp, vp]),
        "ms_precond_build": (C.c_int, [vp, C.POINTER(PrecondOpts), C.POINTER(vp)]),
        "ms_precond_destroy": (C.c_int, [vp]),
        "ms_precond_apply": (C.c_int, [vp, vp, vp]),
        "ms_precond_apply_coarse": (C.c_int, [vp, vp, vp]),
        "ms_precond_info_get": (C.c_int, [vp, C.POINTER(PrecondInfo), ip, dp]),
        "ms_precond_coarse_matrix": (C.c_int, [vp, dp]),
        "ms_pcg_solve": (C.c_int, [vp, vp, vp, C.c_double, C.c_int, vp, C.POINTER(Report), dp, dp, dp]),
        "ms_ctx_set_profiling": (C.c_int, [vp, C.c_int]),
        "ms_ctx_set_profiling_mask": (C.c_int, [vp, C.c_uint]),
        "ms_ctx_profile_get": (C.c_int, [vp, dp, C.POINTER(C.c_longlong)]),
        "ms_ctx_stream": (C.c_void_p, [vp]),
        "ms_precond_bench": (C.c_int, [vp, C.c_int, dp]),
        "ms_nccl_unique_id": (C.c_int, [C.c_char_p]),
        "ms_ctx_attach_nccl": (C.c_int, [vp, C.c_int, C.c_int, C.c_char_p]),
        "ms_ctx_attach_callbacks": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(CommCallbacks)]),
        "ms_comm_selftest": (C.c_int, [vp, dp]),
        "ms_strip_rows": (C.c_int, [C.c_int, C.c_int, C.c_int, ip, ip]),
        "ms_copy": (C.c_int, [vp, vp, C.c_size_t]),
        "ms_cache_trim": (C.c_int, [C.c_int, C.POINTER(C.c_size_t)]),
        "ms_halo_plan": (C.c_int, [C.c_int] * 6 + [ip]),
        "ms_filter_create": (C.c_int, [vp, C.c_int, C.c_int, C.c_double, C.c_double, C.POINTER(vp)]),
        "ms_filter_destroy": (C.c_int, [vp]),
        "ms_filter_apply": (C.c_int, [vp, vp, vp]),
        "ms_filter_adjoint": (C.c_int, [vp, vp, vp]),
        "ms_problem_set_density": (C.c_int, [vp, vp, C.c_double, C.c_double, C.c_double]),
        "ms_compliance_sensitivity": (C.c_int, [vp, C.c_int, C.c_int, C.c_double, vp, vp, vp, C.c_double,
                                                C.c_double, C.c_double, dp, vp]),
        "ms_oc_update": (C.c_int, [vp, C.c_int64, vp, vp, vp, vp, C.c_double, C.c_double, C.c_double, vp, ip]),
        "ms_dot": (C.c_int, [vp, C.c_int64, vp, vp, dp]),
        "ms_unit_element": (C.c_int, [C.c_double, dp]),
        "ms_dense_spd_solve": (C.c_int, [vp, C.c_int, vp, vp, vp, C.c_int]),
        "ms_csr_create": (C.c_int, [vp, C.c_int64, i64p, ip, dp, C.POINTER(vp)]),
        "ms_csr_apply": (C.c_int, [vp, vp, vp]),
        "ms_csr_destroy": (C.c_int, [vp]),
        "ms_pcg_solve_generic": (C.c_int, [vp, C.c_int64, C.POINTER(LinOp), C.POINTER(LinOp), vp, C.c_double,
                                           C.c_int, vp, C.POINTER(Report), dp, dp, dp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(code, ctx=None):
    """Map ABI status codes onto the reference's exception types."""
    if code == MS_OK:
        return
    buf = C.create_string_buffer(2048)
    load().ms_last_error(ctx, buf, len(buf))
    msg = buf.value.decode(errors="replace") or f"msgpu error {code}"
    if code in (MS_E_INVALID, MS_E_NOT_SPD):
        raise ValueError(msg)
    if code == MS_E_NOMEM:
        raise MemoryError(msg)
    raise MsError(msg)


def vec_ptr(a):
    """(pointer, keepalive, is_device) for a float64 numpy array or torch CUDA tensor."""
    mod = type(a).__module__
    if mod.startswith("torch"):
        import torch

        if a.dtype != torch.float64:
            raise TypeError("expected a float64 tensor")
        t = a.contiguous()
        if t.is_cuda:
            torch.cuda.synchronize(t.device)
        return C.c_void_p(t.data_ptr()), t, t.is_cuda
    arr = np.ascontiguousarray(a, dtype=np.float64)
    return C.c_void_p(arr.ctypes.data), arr, False


def dptr(arr):
    return arr.ctypes.data_as(C.POINTER(C.c_double))


def iptr(arr):
    return arr.ctypes.data_as(C.POINTER(C.c_int))


def cache_trim(release=False):
    """Bytes of device memory held by the library's block cache on the current
    device (released buffers kept for reuse); with release=True they are first
    returned to the driver (ms_cache_trim)."""
    out = C.c_size_t(0)
    check(load().ms_cache_trim(1 if release else 0, C.byref(out)))
    return int(out.value)
