"""Device-side problem generation (csrc/generate.cu).

``DeviceMatrix.generate`` assembles a stencil matrix directly in HBM
(bit-identical to the host ``stencil``); it can stand wherever the API takes a
matrix on that context (``bcg_solve``, ``bop``, ``DeviceSolver``) and
``download()`` returns the host ``SparseMatrix``.  ``DeviceSolver.generate_rhs``
fills the resident right hand side on the device.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _native as N
from .blockkrylov import ConfigError, Context, SparseMatrix, _check, default_context


class DeviceMatrix:
    """A matrix that lives on one context's device only (bkg_matrix_generate)."""

    def __init__(self, handle: C.c_void_p, n: int, nnz: int, ctx: Context):
        self.handle, self._n, self._nnz, self.ctx = handle, n, nnz, ctx

    @staticmethod
    def generate(kind: int, nx: int, ny: int, nz: int = 1, seed: int = 0, contrast: float = 2.0,
                 ctx: Optional[Context] = None) -> "DeviceMatrix":
        """Stencil kinds of ``stencil`` (0 poisson2d constant, 1 log-uniform,
        2 exp(N(0,1)) diffusion, 3 3D 7-point, 4 3D 27-point)."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(N.lib().bkg_matrix_generate(ctx.handle, kind, nx, ny, nz, seed, float(contrast),
                                           C.byref(h)))
        n, nnz = C.c_uint64(), C.c_uint64()
        _check(N.lib().bkg_matrix_info(h, C.byref(n), C.byref(nnz)))
        m = DeviceMatrix(h, int(n.value), int(nnz.value), ctx)
        ctx.adopt(m)
        return m

    def n(self) -> int:
        return self._n

    def nnz(self) -> int:
        return self._nnz

    def device(self, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        if ctx is not self.ctx:
            raise ConfigError("DeviceMatrix: generated on another context")
        return self.handle

    def download(self) -> SparseMatrix:
        rp = np.empty(self._n + 1, dtype=np.uint64)
        cl = np.empty(self._nnz, dtype=np.uint64)
        vl = np.empty(self._nnz, dtype=np.float64)
        _check(N.lib().bkg_matrix_download(self.handle, rp.ctypes.data_as(C.POINTER(C.c_uint64)),
                                           cl.ctypes.data_as(C.POINTER(C.c_uint64)),
                                           vl.ctypes.data_as(C.POINTER(C.c_double))))
        return SparseMatrix(self._n, rp, cl, vl, validate=False)

    def close(self) -> None:
        if self.handle:
            N.lib().bkg_matrix_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
