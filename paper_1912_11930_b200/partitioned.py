"""Row-partitioned Block-CG (multi-GPU path) over bkg_psolver_*.

The rows of A are split into contiguous blocks; each block ("part") owns its
rows of X, R, Q and a ghost-extended P.  Two transports share one code path:

* ``PartitionedSolver.virtual(a, cfg, nparts)`` — all parts on this process's
  device (halo = device copies, allreduce = fixed-order sum kernel): the
  single-GPU emulation of ``nparts`` ranks used by the tests;
* ``PartitionedSolver.nccl(...)`` — one part per process (torchrun rank), halo
  with ncclSend/ncclRecv over NVLink, ncclAllReduce of the Gram partials.

``halo_plan`` / ``need_range`` are the pure host logic (no GPU needed).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Tuple

import numpy as np

from . import _native as N
from .blockkrylov import Context, SparseMatrix, SubalgebraConfig, _check, _dp, _up, default_context


def row_blocks(n: int, nparts: int) -> List[int]:
    """Contiguous near-equal row blocks [b[r], b[r+1]) (same split as the C ABI)."""
    return [n * r // nparts for r in range(nparts + 1)]


def local_csr(a: SparseMatrix, r0: int, r1: int):
    """Rows [r0, r1) of A: (local row offsets from 0, global columns, values)."""
    off = a.row_offsets()
    s, e = int(off[r0]), int(off[r1])
    lrp = (off[r0:r1 + 1] - off[r0]).astype(np.uint64)
    return lrp, a.col_indices()[s:e].copy(), a.values()[s:e].copy()


def need_range(r0: int, r1: int, cols: np.ndarray) -> Tuple[int, int]:
    """Operand rows a part touches: [min(r0, min col), max(r1, max col + 1))."""
    if cols.size == 0:
        return r0, r1
    return min(r0, int(cols.min())), max(r1, int(cols.max()) + 1)


def halo_plan(row_begin, need_lo, need_hi) -> List[Tuple[int, int, int, int]]:
    """(dst part, src part, first global row, rows) copies (bkg_halo_plan)."""
    nparts = len(need_lo)
    rb = np.ascontiguousarray(row_begin, dtype=np.int64)
    lo = np.ascontiguousarray(need_lo, dtype=np.int64)
    hi = np.ascontiguousarray(need_hi, dtype=np.int64)
    cap = nparts * nparts
    out = np.zeros(4 * max(cap, 1), dtype=np.int64)
    cnt = C.c_uint64()
    p64 = C.POINTER(C.c_int64)
    _check(N.lib().bkg_halo_plan(nparts, rb.ctypes.data_as(p64), lo.ctypes.data_as(p64),
                                 hi.ctypes.data_as(p64), out.ctypes.data_as(p64), cap,
                                 C.byref(cnt)))
    return [tuple(int(v) for v in out[4 * i:4 * i + 4]) for i in range(cnt.value)]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(N.lib().bkg_nccl_unique_id(buf))
    return buf.raw


class PartitionedSolver:
    def __init__(self, handle, ctx: Context, n: int, k: int, rows: Tuple[int, int], virtual: bool):
        self.handle, self.ctx, self.n, self.k = handle, ctx, n, k
        ctx.adopt(self)
        self.rows = rows
        self.is_virtual = virtual

    @staticmethod
    def virtual(a: SparseMatrix, cfg: SubalgebraConfig, nparts: int,
                ctx: Optional[Context] = None) -> "PartitionedSolver":
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(N.lib().bkg_psolver_create_virtual(ctx.handle, a.n(), _up(a.row_offsets()),
                                                  _up(a.col_indices()), _dp(a.values()), nparts,
                                                  cfg.k, cfg.p, cfg._mode_code, C.byref(h)))
        return PartitionedSolver(h, ctx, a.n(), cfg.k, (0, a.n()), True)

    @staticmethod
    def nccl(n_global: int, r0: int, r1: int, lrowptr, cols, vals, cfg: SubalgebraConfig,
             rank: int, nranks: int, nccl_id: bytes,
             ctx: Optional[Context] = None) -> "PartitionedSolver":
        ctx = ctx or default_context()
        lrowptr = np.ascontiguousarray(lrowptr, dtype=np.uint64)
        cols = np.ascontiguousarray(cols, dtype=np.uint64)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        h = C.c_void_p()
        idb = C.create_string_buffer(nccl_id, 128)
        _check(N.lib().bkg_psolver_create_nccl(ctx.handle, n_global, r0, r1, _up(lrowptr),
                                               _up(cols), _dp(vals), cfg.k, cfg.p,
                                               cfg._mode_code, rank, nranks, idb, C.byref(h)))
        return PartitionedSolver(h, ctx, n_global, cfg.k, (r0, r1), False)

    @staticmethod
    def nccl_generated(kind: int, nx: int, ny: int, nz: int, r0: int, r1: int,
                       cfg: SubalgebraConfig, rank: int, nranks: int, nccl_id: bytes,
                       ctx: Optional[Context] = None, rhs: Optional[str] = "normal",
                       seed: int = 7, coeff_seed: int = 0,
                       contrast: float = 2.0) -> "PartitionedSolver":
        """One rank's rows [r0, r1) of a stencil matrix generated on its own
        device (bkg_psolver_create_nccl_generated); B's rows generated there
        too when rhs is "normal" / "uniform" (bkg_psolver_generate_rhs)."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        idb = C.create_string_buffer(nccl_id, 128)
        _check(N.lib().bkg_psolver_create_nccl_generated(
            ctx.handle, kind, nx, ny, nz, coeff_seed, contrast, r0, r1, cfg.k, cfg.p,
            cfg._mode_code, rank, nranks, idb, C.byref(h)))
        n = nx * ny * (nz if kind >= 3 else 1)
        s = PartitionedSolver(h, ctx, n, cfg.k, (r0, r1), False)
        if rhs is not None:
            s.generate_rhs(rhs, seed)
        return s

    def generate_rhs(self, distribution: str = "normal", seed: int = 7) -> None:
        d = {"uniform": 0, "normal": 1}[distribution]
        _check(N.lib().bkg_psolver_generate_rhs(self.handle, d, seed))

    def rhs(self) -> np.ndarray:
        rows = self.rows[1] - self.rows[0]
        out = np.empty((rows, self.k))
        _check(N.lib().bkg_psolver_get_rhs(self.handle, _dp(out)))
        return out

    def set_rhs(self, b: np.ndarray) -> None:
        b = np.ascontiguousarray(b, dtype=np.float64)
        _check(N.lib().bkg_psolver_set_rhs(self.handle, _dp(b)))

    def run(self, tol: float = 1e-8, max_iter: int = 0, record_history: bool = False,
            final_norms: bool = False):
        rep = N.Report()
        fin = np.zeros(self.k)
        _check(N.lib().bkg_psolver_run(self.handle, tol, max_iter, int(record_history),
                                       _dp(fin) if final_norms else None, C.byref(rep)))
        return rep, fin

    def x(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        rows = self.rows[1] - self.rows[0]
        if out is None:
            out = np.empty((rows, self.k))
        assert out.shape == (rows, self.k) and out.dtype == np.float64 and out.flags.c_contiguous
        _check(N.lib().bkg_psolver_get_x(self.handle, _dp(out)))
        return out

    def history(self, cap: int) -> np.ndarray:
        out = np.empty((max(cap, 1), self.k))
        rows = C.c_uint64()
        _check(N.lib().bkg_psolver_history(self.handle, _dp(out), cap, C.byref(rows)))
        return out[: min(cap, rows.value)]

    def part_info(self, part: int = 0) -> dict:
        """K1 of a part and its interior / boundary block split
        (bkg_psolver_part_info)."""
        out = (C.c_int64 * 9)()
        _check(N.lib().bkg_psolver_part_info(self.handle, part, out))
        from .blockkrylov import Context
        return {"k1": Context.K1_VARIANTS[int(out[0])], "interior_blocks": int(out[1]),
                "boundary_blocks": int(out[2]), "rows": (int(out[3]), int(out[4])),
                "block_rows": int(out[5]), "box": (int(out[6]), int(out[7]), int(out[8]))}

    def close(self) -> None:
        if self.handle:
            N.lib().bkg_psolver_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
