"""ctypes binding of libbkgpu.so (include/bkg.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1912_11930_b200/csrc``).  Loading fails loudly when it is
missing: there is no CPU fallback for the hot path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# BKG_LIB overrides the library path (kernel-variant sweeps in tools/).
LIB_PATH = os.environ.get("BKG_LIB") or os.path.join(HERE, "_build", "libbkgpu.so")

BKG_OK = 0
BKG_DIMENSION = 1
BKG_CONFIG = 2
BKG_BREAKDOWN = 3
BKG_CUDA = 4
BKG_NCCL = 5
BKG_FACTORIZATION = 6
BKG_INTERNAL = 7

BKG_HYBRID = 0
BKG_GLOBAL = 1
BKG_NUMERICS_FAST = 0
BKG_NUMERICS_EXACT = 1

_d = C.POINTER(C.c_double)
_u = C.POINTER(C.c_uint64)
_vp = C.c_void_p


class Report(C.Structure):
    """bkg_report (include/bkg.h) — SolveReport, solver.hpp:48-59."""

    _fields_ = [
        ("iterations", C.c_uint64),
        ("converged", C.c_int32),
        ("breakdown", C.c_int32),
        ("breakdown_iteration", C.c_uint64),
        ("breakdown_block", C.c_uint64),
        ("flops_bdot", C.c_uint64),
        ("flops_baxpy", C.c_uint64),
        ("flops_bop", C.c_uint64),
        ("flops_precond", C.c_uint64),
        ("seconds_bdot", C.c_double),
        ("seconds_baxpy", C.c_double),
        ("seconds_bop", C.c_double),
        ("seconds_precond", C.c_double),
        ("history_rows", C.c_uint64),
        ("loop_seconds", C.c_double),
    ]


ITERATE_FN = C.CFUNCTYPE(None, C.c_uint64, _d, _d, C.c_uint64, C.c_uint64, C.c_void_p)


class SolveOptions(C.Structure):
    _fields_ = [
        ("tol", C.c_double),
        ("max_iter", C.c_uint64),
        ("record_history", C.c_int32),
        ("precond", C.c_int32),
        ("on_iterate", ITERATE_FN),
        ("user", C.c_void_p),
        ("time_kernels", C.c_int32),
    ]


# (name, restype, argtypes) for every symbol declared in include/bkg.h
SIGNATURES = [
    ("bkg_last_error", C.c_char_p, []),
    ("bkg_version", C.c_char_p, []),
    ("bkg_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("bkg_ctx_create", C.c_int, [C.c_int, C.POINTER(_vp)]),
    ("bkg_ctx_destroy", C.c_int, [_vp]),
    ("bkg_ctx_set_numerics", C.c_int, [_vp, C.c_int]),
    ("bkg_ctx_get_numerics", C.c_int, [_vp, C.POINTER(C.c_int)]),
    ("bkg_ctx_stream", C.c_int, [_vp, C.POINTER(_vp)]),
    ("bkg_ctx_launch_count", C.c_int, [_vp, _u]),
    ("bkg_matrix_create", C.c_int, [_vp, C.c_uint64, _u, _u, _d, C.POINTER(_vp)]),
    ("bkg_matrix_destroy", C.c_int, [_vp]),
    ("bkg_matrix_info", C.c_int, [_vp, _u, _u]),
    ("bkg_matrix_generate", C.c_int, [_vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                      C.c_uint64, C.c_double, C.POINTER(_vp)]),
    ("bkg_matrix_download", C.c_int, [_vp, _u, _u, _d]),
    ("bkg_bdot", C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _d, _d, _d, _u]),
    ("bkg_baxpy", C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _d, _d, _d, _u]),
    ("bkg_bop", C.c_int, [_vp, _vp, C.c_uint64, _d, _d, _u]),
    ("bkg_bsolve", C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_int, _d, _d, _d, _u]),
    ("bkg_column_norms", C.c_int, [_vp, C.c_uint64, C.c_uint64, _d, _d]),
    ("bkg_precond_apply", C.c_int, [_vp, _vp, C.c_int, C.c_uint64, _d, _d, _u]),
    ("bkg_precond_setup", C.c_int, [_vp, _vp, C.c_int, C.POINTER(C.c_int64)]),
    ("bkg_solve", C.c_int, [_vp, _vp, C.c_uint64, C.c_uint64, C.c_int, _d, _d,
                            C.POINTER(SolveOptions), _d, _d, C.c_uint64, _d, C.POINTER(Report)]),
    ("bkg_solver_create", C.c_int, [_vp, _vp, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(_vp)]),
    ("bkg_solver_destroy", C.c_int, [_vp]),
    ("bkg_solver_set_rhs", C.c_int, [_vp, _d]),
    ("bkg_solver_generate_rhs", C.c_int, [_vp, C.c_int, C.c_uint64]),
    ("bkg_solver_get_rhs", C.c_int, [_vp, _d]),
    ("bkg_solver_run", C.c_int, [_vp, C.c_double, C.c_uint64, C.c_int, C.POINTER(Report)]),
    ("bkg_solver_get_x", C.c_int, [_vp, _d]),
    ("bkg_solver_history", C.c_int, [_vp, _d, C.c_uint64, _u]),
    ("bkg_solve_history", C.c_int, [_vp, _d, C.c_uint64, _u]),
    ("bkg_solve_k1_variant", C.c_int, [_vp, C.POINTER(C.c_int)]),
    ("bkg_solver_k1_variant", C.c_int, [_vp, C.POINTER(C.c_int)]),
    ("bkg_solver_profile", C.c_int, [_vp, C.c_uint64, _d]),
    ("bkg_solver_debug_first_step", C.c_int, [_vp, _d, _d]),
    ("bkg_solver_kernel_bytes", C.c_int, [_vp, _d]),
    ("bkg_grid_plan", C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int, C.c_int,
                                C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64)]),
    ("bkg_halo_plan", C.c_int, [C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_uint64, _u]),
    ("bkg_nccl_unique_id", C.c_int, [C.c_void_p]),
    ("bkg_psolver_create_virtual", C.c_int, [_vp, C.c_uint64, _u, _u, _d, C.c_int, C.c_uint64,
                                             C.c_uint64, C.c_int, C.POINTER(_vp)]),
    ("bkg_psolver_create_nccl", C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_uint64, _u, _u, _d,
                                          C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                          C.c_void_p, C.POINTER(_vp)]),
    ("bkg_psolver_create_nccl_generated", C.c_int,
     [_vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
      C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_void_p,
      C.POINTER(C.c_void_p)]),
    ("bkg_psolver_generate_rhs", C.c_int, [_vp, C.c_int, C.c_uint64]),
    ("bkg_psolver_get_rhs", C.c_int, [_vp, _d]),
    ("bkg_psolver_part_info", C.c_int, [_vp, C.c_int, C.POINTER(C.c_int64)]),
    ("bkg_psolver_destroy", C.c_int, [_vp]),
    ("bkg_psolver_set_rhs", C.c_int, [_vp, _d]),
    ("bkg_psolver_run", C.c_int, [_vp, C.c_double, C.c_uint64, C.c_int, _d, C.POINTER(Report)]),
    ("bkg_psolver_get_x", C.c_int, [_vp, _d]),
    ("bkg_psolver_history", C.c_int, [_vp, _d, C.c_uint64, _u]),
    ("bkg_stencil_size", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, _u, _u]),
    ("bkg_stencil_fill", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                   C.c_double, _u, _u, _d]),
    ("bkg_random_block_rhs", C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, _d]),
    ("bkg_normal_block_rhs", C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, _d]),
]

_lib = None


def lib() -> C.CDLL:
    """Load libbkgpu.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() — the Block-CG "
                "hot path has no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    msg = lib().bkg_last_error()
    return msg.decode() if msg else ""
