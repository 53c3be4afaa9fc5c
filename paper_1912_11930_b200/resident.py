"""Device-resident Block-CG solver (bkg_solver_*): A, B, X and the work block
vectors stay in HBM between solves.  Used by bench.py for the kernel-only
`value` and the per-kernel roofline; the drop-in call is blockkrylov.bcg_solve.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _native as N
from .blockkrylov import (Context, SparseMatrix, SubalgebraConfig, _check, _dp, default_context)


class DeviceSolver:
    def __init__(self, a, cfg: SubalgebraConfig, ctx: Optional[Context] = None):
        """a: SparseMatrix, or a DeviceMatrix generated on ctx."""
        self.ctx = ctx or default_context()
        self.a, self.cfg = a, cfg
        h = C.c_void_p()
        _check(N.lib().bkg_solver_create(self.ctx.handle, a.device(self.ctx), cfg.k, cfg.p,
                                         cfg._mode_code, C.byref(h)))
        self.handle = h
        self.ctx.adopt(self)

    def set_rhs(self, b: np.ndarray) -> None:
        b = np.ascontiguousarray(b, dtype=np.float64)
        _check(N.lib().bkg_solver_set_rhs(self.handle, _dp(b)))

    def rhs(self) -> np.ndarray:
        """The resident right hand side B (after set_rhs / generate_rhs)."""
        out = np.empty((self.a.n(), self.cfg.k))
        _check(N.lib().bkg_solver_get_rhs(self.handle, _dp(out)))
        return out

    def generate_rhs(self, distribution: str = "uniform", seed: int = 7) -> None:
        """B generated on the device: "uniform" = random_block_rhs(n, k, seed)
        bit for bit, "normal" = the N(0,1) stream within a few ulp."""
        code = {"uniform": 0, "normal": 1}[distribution]
        _check(N.lib().bkg_solver_generate_rhs(self.handle, code, seed))

    def k1(self) -> str:
        """K1 kernel this solver runs (bkg_solver_k1_variant)."""
        v = C.c_int()
        _check(N.lib().bkg_solver_k1_variant(self.handle, C.byref(v)))
        return Context.K1_VARIANTS[v.value]

    def run(self, tol: float = 1e-8, max_iter: int = 0, record_history: bool = False) -> N.Report:
        rep = N.Report()
        _check(N.lib().bkg_solver_run(self.handle, tol, max_iter, int(record_history),
                                      C.byref(rep)))
        return rep

    def x(self) -> np.ndarray:
        out = np.empty((self.a.n(), self.cfg.k))
        _check(N.lib().bkg_solver_get_x(self.handle, _dp(out)))
        return out

    def history(self, cap: int) -> np.ndarray:
        out = np.empty((max(cap, 1), self.cfg.k))
        rows = C.c_uint64()
        _check(N.lib().bkg_solver_history(self.handle, _dp(out), cap, C.byref(rows)))
        return out[: min(cap, rows.value)]

    def profile(self, iterations: int = 20) -> np.ndarray:
        """Average ms per launch of [K1, K2, K3, whole iteration]."""
        out = np.zeros(4)
        _check(N.lib().bkg_solver_profile(self.handle, iterations, _dp(out)))
        return out

    def debug_first_step(self):
        """(Q = A B, [lambda^1 | rho_prev^1]) from one K1 launch (test hook)."""
        q = np.empty((self.a.n(), self.cfg.k))
        cs = self.cfg.block_count() * self.cfg.p ** 2
        coef = np.empty(2 * cs)
        _check(N.lib().bkg_solver_debug_first_step(self.handle, _dp(q), _dp(coef)))
        return q, coef

    def kernel_bytes(self) -> np.ndarray:
        out = np.zeros(4)
        _check(N.lib().bkg_solver_kernel_bytes(self.handle, _dp(out)))
        return out

    def close(self) -> None:
        if self.handle:
            N.lib().bkg_solver_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
