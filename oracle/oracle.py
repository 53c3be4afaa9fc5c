"""ctypes front-end for the CPU oracle — TEST INFRASTRUCTURE ONLY.

Loads either the plain-C restatement (``oracle/liboracle.so``, kind "port")
or the unmodified reference compiled from /root/reference
(``oracle/_ref/libbkref.so``, kind "reference").  Both export the same
signatures (prefix ``orc_`` / ``bkref_``).  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs may import this module; the product package
never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libbkref.so")

POISSON2D_CONST = 0
POISSON2D_LOGUNI = 1
DIFFUSION2D_LOGNORMAL = 2
LAPLACE3D_7PT = 3
STENCIL3D_27PT = 4

PRECOND = {"identity": 0, "jacobi": 1, "ilu0": 2}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_u64 = C.c_uint64


class Report(C.Structure):
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
    ]


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


@dataclass
class SolveOut:
    x: np.ndarray
    history: np.ndarray
    final_norms: np.ndarray
    report: Report


class Oracle:
    """One CPU implementation of the path (port or reference)."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        p = "orc_" if kind == "port" else "bkref_"
        self.p = p
        L = self.lib
        self._f = lambda name: getattr(L, p + name)
        f = self._f
        f("rng_symmetric").argtypes = [_u64, _sz, _dp]
        f("random_block_rhs").argtypes = [_sz, _sz, _u64, _dp]
        f("bdot").argtypes = [_sz, _sz, _sz, C.c_int, _dp, _dp, _dp]
        f("baxpy").argtypes = [_sz, _sz, _sz, C.c_int, _dp, _dp, _dp]
        f("bop").argtypes = [_sz, _up, _up, _dp, _sz, _dp, _dp]
        f("bsolve").argtypes = [_sz, _sz, C.c_int, _dp, _dp, _dp, C.POINTER(C.c_uint64)]
        f("bsolve").restype = C.c_int
        f("column_norms").argtypes = [_sz, _sz, _dp, _dp]
        f("bcg_solve").argtypes = [
            _sz, _up, _up, _dp, C.c_int, _sz, _sz, C.c_int, _dp, C.c_void_p, C.c_double,
            _u64, C.c_int, C.c_void_p, _u64, _dp, _dp, C.POINTER(Report)]
        f("bcg_solve").restype = C.c_int
        f("bench_solve").argtypes = [C.c_int, _sz, _up, _up, _dp, _sz, _sz, C.c_int, _dp,
                                     C.c_double, _u64, C.POINTER(C.c_uint64)]
        f("bench_solve").restype = C.c_double
        if kind == "reference":
            L.bkref_bench_iterations.argtypes = [C.c_int, _sz, _up, _up, _dp, _sz, _sz, C.c_int,
                                                 _dp, _u64, C.POINTER(C.c_uint64)]
            L.bkref_bench_iterations.restype = C.c_double
        if kind == "port":
            L.orc_normal_block_rhs.argtypes = [_sz, _sz, _u64, _dp]
            L.orc_stencil_nnz.argtypes = [C.c_int, _sz, _sz, _sz]
            L.orc_stencil_nnz.restype = _sz
            L.orc_stencil_rows.argtypes = [C.c_int, _sz, _sz, _sz]
            L.orc_stencil_rows.restype = _sz
            L.orc_stencil_fill.argtypes = [C.c_int, _sz, _sz, _sz, _u64, C.c_double, _up, _up,
                                           _dp]
            L.orc_stencil_fill.restype = C.c_int
        else:
            L.bkref_poisson2d.argtypes = [_sz, _sz, _u64, C.c_double, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
            L.bkref_poisson2d.restype = _sz

    # ---- generators -------------------------------------------------
    def rng_symmetric(self, seed, count):
        out = np.empty(count)
        self._f("rng_symmetric")(seed, count, out)
        return out

    def random_block_rhs(self, n, k, seed):
        out = np.empty((n, k))
        self._f("random_block_rhs")(n, k, seed, out)
        return out

    def normal_block_rhs(self, n, k, seed):
        out = np.empty((n, k))
        self.lib.orc_normal_block_rhs(n, k, seed, out)
        return out

    def stencil(self, kind, nx, ny, nz=1, seed=0, contrast=2.0):
        """CSR (rowptr, cols, vals) as uint64/uint64/float64 arrays."""
        if self.kind == "reference":
            assert kind in (POISSON2D_CONST, POISSON2D_LOGUNI)
            c = -1.0 if kind == POISSON2D_CONST else contrast
            nnz = self.lib.bkref_poisson2d(nx, ny, seed, c, None, None, None)
            n = nx * ny
            rp = np.empty(n + 1, np.uint64)
            cols = np.empty(nnz, np.uint64)
            vals = np.empty(nnz)
            self.lib.bkref_poisson2d(nx, ny, seed, c, rp.ctypes.data, cols.ctypes.data,
                                     vals.ctypes.data)
            return rp, cols, vals
        n = self.lib.orc_stencil_rows(kind, nx, ny, nz)
        nnz = self.lib.orc_stencil_nnz(kind, nx, ny, nz)
        rp = np.empty(n + 1, np.uint64)
        cols = np.empty(nnz, np.uint64)
        vals = np.empty(nnz)
        st = self.lib.orc_stencil_fill(kind, nx, ny, nz, seed, contrast, rp, cols, vals)
        if st != 0:
            raise ValueError("stencil_fill failed")
        assert rp[-1] == nnz
        return rp, cols, vals

    # ---- kernels ------------------------------------------------------
    def bdot(self, x, y, p, glob=False):
        n, k = x.shape
        blocks = 1 if glob else k // p
        out = np.empty((blocks, p, p))
        self._f("bdot")(n, k, p, int(glob), np.ascontiguousarray(x), np.ascontiguousarray(y),
                        out)
        return out

    def baxpy(self, x, y, gamma, p, glob=False):
        x = np.array(x, dtype=np.float64, order="C", copy=True)
        n, k = x.shape
        self._f("baxpy")(n, k, p, int(glob), x, np.ascontiguousarray(y),
                         np.ascontiguousarray(gamma, dtype=np.float64))
        return x

    def bop(self, csr, x):
        rp, cols, vals = csr
        n, k = x.shape
        y = np.empty_like(x)
        self._f("bop")(n, rp, cols, vals, k, np.ascontiguousarray(x), y)
        return y

    def bsolve(self, gamma, delta, k, p, glob=False):
        out = np.empty_like(np.ascontiguousarray(delta, dtype=np.float64))
        bad = C.c_uint64(0)
        st = self._f("bsolve")(k, p, int(glob), np.ascontiguousarray(gamma, dtype=np.float64),
                               np.ascontiguousarray(delta, dtype=np.float64), out, C.byref(bad))
        return out, (None if st == 0 else int(bad.value))

    def column_norms(self, x):
        n, k = x.shape
        out = np.empty(k)
        self._f("column_norms")(n, k, np.ascontiguousarray(x), out)
        return out

    def bcg_solve(self, csr, b, p, glob=False, x0=None, tol=1e-8, max_iter=0,
                  record_history=True, precond="identity", history_cap=None):
        rp, cols, vals = csr
        n, k = b.shape
        b = np.ascontiguousarray(b)
        x = np.empty_like(b)
        fin = np.empty(k)
        cap = history_cap if history_cap is not None else (max_iter or 10 * n) + 1
        cap = min(cap, 1 << 22)
        hist = np.zeros((cap, k)) if record_history else np.zeros((1, k))
        rep = Report()
        x0p = None
        if x0 is not None:
            x0 = np.ascontiguousarray(x0, dtype=np.float64)
            x0p = x0.ctypes.data
        st = self._f("bcg_solve")(n, rp, cols, vals, PRECOND[precond], k, p, int(glob), b, x0p,
                                  tol, max_iter, int(record_history), hist.ctypes.data,
                                  cap if record_history else 0, x, fin, C.byref(rep))
        if st != 0:
            raise ValueError(f"oracle bcg_solve status {st}")
        rows = min(rep.history_rows, cap) if record_history else 0
        return SolveOut(x, hist[:rows].copy(), fin, rep)

    def bench_solve(self, threads, csr, b, p, glob, tol, max_iter):
        rp, cols, vals = csr
        n, k = b.shape
        its = C.c_uint64(0)
        dt = self._f("bench_solve")(threads, n, rp, cols, vals, k, p, int(glob),
                                    np.ascontiguousarray(b), tol, max_iter, C.byref(its))
        return dt, int(its.value)


    def bench_iterations(self, threads, csr, b, p, glob, iters):
        """Reference only: seconds of `threads` concurrent solves' iterations
        1..iters, setup and final residual excluded (observer-timed)."""
        rp, cols, vals = csr
        n, k = b.shape
        its = C.c_uint64(0)
        dt = self.lib.bkref_bench_iterations(threads, n, rp, cols, vals, k, p, int(glob),
                                             np.ascontiguousarray(b), iters, C.byref(its))
        return dt, int(its.value)


def available(kind: str) -> bool:
    return os.path.exists(PORT_LIB if kind == "port" else REF_LIB)
