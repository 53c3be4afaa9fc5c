"""Host-side mirror of the reference ``blockkrylov`` C++ API, over the C ABI.

Names, argument meaning and error behaviour follow the reference headers in
``proj/include/blockkrylov`` (cited per symbol) so that code and tests written
against the reference read the same here.  Block vectors are NumPy arrays of
shape (n, k), float64, C order — exactly the reference's lane-interleaved
``data[row * k + col]`` layout (block_vector.hpp:18-21).  Every arithmetic
step runs on the GPU through ``libbkgpu.so``; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import itertools
import weakref
import os
import threading
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _native as N

# --------------------------------------------------------------- errors ----
class Error(RuntimeError):
    """blockkrylov::Error (errors.hpp:10-13)."""


class DimensionError(Error):
    """errors.hpp:16-19."""


class ConfigError(Error):
    """errors.hpp:22-25."""


class SizeError(Error):
    """errors.hpp:28-31."""


class BreakdownError(Error):
    """errors.hpp:34-43 — carries the singular block's index."""

    def __init__(self, block_index: int, what: str):
        super().__init__(what)
        self.block_index = block_index


class FactorizationError(Error):
    """errors.hpp:46-55."""

    def __init__(self, row: int, what: str):
        super().__init__(what)
        self.row = row


class CudaError(Error):
    """Device failure (no reference counterpart)."""


def _check(status: int, **extra) -> None:
    if status == N.BKG_OK:
        return
    msg = N.last_error()
    if status == N.BKG_DIMENSION:
        raise DimensionError(msg)
    if status == N.BKG_CONFIG:
        raise ConfigError(msg)
    if status == N.BKG_BREAKDOWN:
        raise BreakdownError(extra.get("block", -1), msg)
    if status == N.BKG_FACTORIZATION:
        raise FactorizationError(extra.get("row", -1), msg)
    if status == N.BKG_CUDA:
        raise CudaError(msg)
    raise Error(f"status {status}: {msg}")


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _up(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


# -------------------------------------------------------------- context ----
class Context:
    """One device + stream + numerics mode (bkg_ctx)."""

    _uids = itertools.count(1)

    def __init__(self, device: int = 0, numerics: str = "fast"):
        h = C.c_void_p()
        _check(N.lib().bkg_ctx_create(device, C.byref(h)))
        self.handle = h
        # cache key for device matrices: handles can be reused after close()
        self.uid = next(Context._uids)
        self._children = weakref.WeakSet()
        self.device = device
        self.set_numerics(numerics)

    def set_numerics(self, numerics: str) -> None:
        mode = {"fast": N.BKG_NUMERICS_FAST, "exact": N.BKG_NUMERICS_EXACT}[numerics]
        _check(N.lib().bkg_ctx_set_numerics(self.handle, mode))
        self.numerics = numerics

    def stream(self) -> int:
        """cudaStream_t (as an int) all launches of this context go to."""
        s = C.c_void_p()
        _check(N.lib().bkg_ctx_stream(self.handle, C.byref(s)))
        return s.value or 0

    def launch_count(self) -> int:
        v = C.c_uint64()
        _check(N.lib().bkg_ctx_launch_count(self.handle, C.byref(v)))
        return v.value

    K1_VARIANTS = {-1: "exact", 0: "k1_wide", 1: "k1_line", 2: "k1_stage", 3: "resident", 4: "k1_grid"}

    def last_k1(self) -> str:
        """K1 kernel of this context's last bcg_solve (bkg_solve_k1_variant)."""
        v = C.c_int()
        _check(N.lib().bkg_solve_k1_variant(self.handle, C.byref(v)))
        return self.K1_VARIANTS[v.value]

    def adopt(self, obj) -> None:
        """Register a native object bound to this context (it is closed first
        when the context closes, so nothing outlives its bkg_ctx)."""
        self._children.add(obj)

    def close(self) -> None:
        if self.handle:
            for obj in list(self._children):
                obj.close()
            N.lib().bkg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


_default: Optional[Context] = None
_lock = threading.Lock()


def default_context() -> Context:
    global _default
    with _lock:
        if _default is None:
            _default = Context(int(os.environ.get("BKG_DEVICE", "0")),
                               os.environ.get("BKG_NUMERICS", "fast"))
        return _default


def set_numerics(numerics: str) -> None:
    """'exact' (bit-identical to the reference) or 'fast' (fused kernels)."""
    default_context().set_numerics(numerics)


# -------------------------------------------------------- subalgebra -------
HYBRID = "hybrid"
GLOBAL = "global"


class SubalgebraConfig:
    """(k, p, mode) with q = k/p (subalgebra.hpp:33-74)."""

    def __init__(self, k: int, p: int, mode: str = HYBRID):
        if k <= 0 or p <= 0:
            raise ConfigError("subalgebra: k and p must be positive")
        if k % p != 0:
            raise ConfigError(f"subalgebra: block width p={p} does not divide k={k}")
        if mode not in (HYBRID, GLOBAL):
            raise ConfigError(f"unknown subalgebra mode '{mode}' (expected hybrid or global)")
        self.k, self.p, self.mode = int(k), int(p), mode
        self.q = self.k // self.p

    @staticmethod
    def classical(k: int) -> "SubalgebraConfig":
        return SubalgebraConfig(k, k, HYBRID)

    @staticmethod
    def parallel(k: int) -> "SubalgebraConfig":
        return SubalgebraConfig(k, 1, HYBRID)

    def block_count(self) -> int:
        return 1 if self.mode == GLOBAL else self.q

    @property
    def _mode_code(self) -> int:
        return N.BKG_GLOBAL if self.mode == GLOBAL else N.BKG_HYBRID

    def __eq__(self, o) -> bool:
        return isinstance(o, SubalgebraConfig) and (self.k, self.p, self.mode) == (o.k, o.p, o.mode)

    def __repr__(self) -> str:
        return f"SubalgebraConfig(k={self.k}, p={self.p}, mode={self.mode})"


class BlockCoefficient:
    """q (hybrid) or 1 (global) dense p x p blocks, row-major (subalgebra.hpp:78-120)."""

    def __init__(self, config: SubalgebraConfig, data: Optional[np.ndarray] = None):
        self.config = config
        shape = (config.block_count(), config.p, config.p)
        if data is None:
            self.data = np.zeros(shape)
        else:
            self.data = np.ascontiguousarray(data, dtype=np.float64).reshape(shape)

    @staticmethod
    def identity(config: SubalgebraConfig) -> "BlockCoefficient":
        c = BlockCoefficient(config)
        for b in range(config.block_count()):
            c.data[b] = np.eye(config.p)
        return c

    def block_count(self) -> int:
        return self.config.block_count()

    def block(self, b: int) -> np.ndarray:
        return self.data[b]

    def entry(self, b: int, row: int, col: int) -> float:
        return float(self.data[b, row, col])

    def negated(self) -> "BlockCoefficient":
        return BlockCoefficient(self.config, -self.data)


@dataclass
class FlopCounter:
    """kernels.hpp:22-32."""

    multiply_adds_bdot: int = 0
    multiply_adds_baxpy: int = 0
    multiply_adds_bop: int = 0
    multiply_adds_precond: int = 0

    def total(self) -> int:
        return (self.multiply_adds_bdot + self.multiply_adds_baxpy + self.multiply_adds_bop +
                self.multiply_adds_precond)


def block_vector(n: int, k: int, value: float = 0.0) -> np.ndarray:
    """BlockVector(n, k, value) (block_vector.hpp:27-30)."""
    if k == 0:
        raise ConfigError("BlockVector: column count must be positive")
    return np.full((n, k), value, dtype=np.float64)


def _bv(x) -> np.ndarray:
    a = np.asarray(x)
    if a.ndim != 2:
        raise DimensionError("block vector must be 2-D (n x k)")
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        a = np.ascontiguousarray(a, dtype=np.float64)
    return a


# --------------------------------------------------------- sparse matrix ---
class SparseMatrix:
    """Symmetric CSR matrix (sparse_matrix.hpp:27-131); validates on construction."""

    def __init__(self, n: int, row_offsets, col_indices, values, validate: bool = True):
        self._n = int(n)
        self.row_offsets_ = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        self.col_indices_ = np.ascontiguousarray(col_indices, dtype=np.uint64)
        self.values_ = np.ascontiguousarray(values, dtype=np.float64)
        self._dev = {}
        if validate:
            self._validate()

    @staticmethod
    def from_triplets(n: int, triplets) -> "SparseMatrix":
        """sparse_matrix.hpp:39-64 — duplicates are summed."""
        t = sorted(((int(r), int(c), float(v)) for r, c, v in triplets), key=lambda e: (e[0], e[1]))
        counts = [0] * n
        cols: List[int] = []
        vals: List[float] = []
        for r, c, v in t:
            if r >= n or c >= n:
                raise ConfigError("triplet index out of range")
            if counts[r] > 0 and cols[-1] == c:
                vals[-1] += v
                continue
            counts[r] += 1
            cols.append(c)
            vals.append(v)
        offsets = np.zeros(n + 1, dtype=np.uint64)
        np.cumsum(counts, out=offsets[1:])
        return SparseMatrix(n, offsets, np.array(cols, dtype=np.uint64), np.array(vals))

    def _validate(self) -> None:  # sparse_matrix.hpp:89-125
        n, off, cols, vals = self._n, self.row_offsets_, self.col_indices_, self.values_
        if n == 0:
            raise ConfigError("sparse matrix: dimension must be positive")
        if off.size != n + 1:
            raise ConfigError("sparse matrix: row_offsets must have n+1 entries")
        if off[0] != 0 or off[-1] != vals.size or cols.size != vals.size:
            raise ConfigError("sparse matrix: offsets inconsistent with stored entries")
        if np.any(off[1:] < off[:-1]):
            raise ConfigError("sparse matrix: row_offsets must be non-decreasing")
        if cols.size and np.any(cols >= n):
            raise ConfigError("sparse matrix: column index out of range")
        rows = np.repeat(np.arange(n, dtype=np.uint64), np.diff(off).astype(np.int64))
        if cols.size > 1:
            same_row = rows[1:] == rows[:-1]
            if np.any(same_row & (cols[1:] <= cols[:-1])):
                raise ConfigError("sparse matrix: columns must be strictly ascending per row")
        keys = rows * np.uint64(n) + cols
        tkeys = cols * np.uint64(n) + rows
        pos = np.searchsorted(keys, tkeys)
        pos_c = np.minimum(pos, max(keys.size - 1, 0))
        found = (pos < keys.size) & (keys[pos_c] == tkeys)
        if not np.all(found):
            bad = int(np.argmin(found))
            raise ConfigError(f"sparse matrix: entry ({int(rows[bad])},{int(cols[bad])}) has no "
                              "symmetric counterpart")
        w = vals[pos_c]
        scale = np.maximum(np.abs(vals), np.abs(w))
        if np.any(np.abs(vals - w) > 1e-14 * scale):
            raise ConfigError("sparse matrix: values not symmetric")

    def n(self) -> int:
        return self._n

    def nnz(self) -> int:
        return int(self.values_.size)

    def row_offsets(self) -> np.ndarray:
        return self.row_offsets_

    def col_indices(self) -> np.ndarray:
        return self.col_indices_

    def values(self) -> np.ndarray:
        return self.values_

    def diagonal(self) -> np.ndarray:
        """A(r, r) for every row (0 where not stored), vectorised."""
        n = self._n
        rows = np.repeat(np.arange(n, dtype=np.uint64), np.diff(self.row_offsets_).astype(np.int64))
        hit = self.col_indices_ == rows
        d = np.zeros(n)
        d[rows[hit].astype(np.int64)] = self.values_[hit]
        return d

    def at(self, row: int, col: int) -> float:
        lo, hi = int(self.row_offsets_[row]), int(self.row_offsets_[row + 1])
        i = lo + int(np.searchsorted(self.col_indices_[lo:hi], col))
        if i < hi and int(self.col_indices_[i]) == col:
            return float(self.values_[i])
        return 0.0

    def device(self, ctx: Optional[Context] = None):
        """Device-resident copy on ctx (uploaded once, cached)."""
        ctx = ctx or default_context()
        key = ctx.uid
        h = self._dev.get(key)
        if h is None:
            h = C.c_void_p()
            _check(N.lib().bkg_matrix_create(ctx.handle, self._n, _up(self.row_offsets_),
                                             _up(self.col_indices_), _dp(self.values_),
                                             C.byref(h)))
            self._dev[key] = h
        return h

    def release_device(self) -> None:
        for h in self._dev.values():
            N.lib().bkg_matrix_destroy(h)
        self._dev.clear()

    def __del__(self):  # pragma: no cover
        try:
            self.release_device()
        except Exception:
            pass

    def __eq__(self, o) -> bool:
        return (isinstance(o, SparseMatrix) and self._n == o._n and
                np.array_equal(self.row_offsets_, o.row_offsets_) and
                np.array_equal(self.col_indices_, o.col_indices_) and
                np.array_equal(self.values_, o.values_))


# ---------------------------------------------------------------- kernels --
def bdot(x, y, cfg: SubalgebraConfig, flops: Optional[FlopCounter] = None,
         ctx: Optional[Context] = None) -> BlockCoefficient:
    """BDOT (kernels.hpp:59-88)."""
    x, y = _bv(x), _bv(y)
    if x.shape != y.shape:
        raise DimensionError(f"bdot: block vectors have shapes {x.shape[0]}x{x.shape[1]} and "
                             f"{y.shape[0]}x{y.shape[1]}")
    if x.shape[1] != cfg.k:
        raise DimensionError(f"bdot: block vector has k={x.shape[1]} but configuration expects "
                             f"k={cfg.k}")
    ctx = ctx or default_context()
    out = BlockCoefficient(cfg)
    f = C.c_uint64(0)
    _check(N.lib().bkg_bdot(ctx.handle, x.shape[0], cfg.k, cfg.p, cfg._mode_code, _dp(x), _dp(y),
                            _dp(out.data), C.byref(f)))
    if flops is not None:
        flops.multiply_adds_bdot += f.value
    return out


def baxpy(x: np.ndarray, y, gamma: BlockCoefficient, flops: Optional[FlopCounter] = None,
          ctx: Optional[Context] = None) -> None:
    """BAXPY X <- X + Y embed(gamma), in place (kernels.hpp:94-125)."""
    if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous):
        raise DimensionError("baxpy: X must be a C-contiguous float64 (n x k) array")
    y = _bv(y)
    if x.shape != y.shape:
        raise DimensionError(f"baxpy: block vectors have shapes {x.shape} and {y.shape}")
    cfg = gamma.config
    if x.ndim != 2 or x.shape[1] != cfg.k:
        raise DimensionError(f"baxpy: block vector has k={x.shape[-1]} but configuration expects "
                             f"k={cfg.k}")
    if x is y or np.shares_memory(x, y):
        raise DimensionError("baxpy: X and Y must be distinct")
    ctx = ctx or default_context()
    f = C.c_uint64(0)
    g = np.ascontiguousarray(gamma.data, dtype=np.float64)
    _check(N.lib().bkg_baxpy(ctx.handle, x.shape[0], cfg.k, cfg.p, cfg._mode_code, _dp(x), _dp(y),
                             _dp(g), C.byref(f)))
    if flops is not None:
        flops.multiply_adds_baxpy += f.value


def bop(a: SparseMatrix, x, y: Optional[np.ndarray] = None, flops: Optional[FlopCounter] = None,
        ctx: Optional[Context] = None) -> np.ndarray:
    """BOP Y = A X (kernels.hpp:129-164); returns Y (allocated when y is None)."""
    x = _bv(x)
    if a.n() != x.shape[0]:
        raise DimensionError(f"bop: matrix is {a.n()}-dimensional but block vector has "
                             f"{x.shape[0]} rows")
    if y is None or y.shape != x.shape or y.dtype != np.float64 or not y.flags.c_contiguous:
        y = np.empty_like(x)
    if y is x:
        raise DimensionError("bop: X and Y must be distinct")
    ctx = ctx or default_context()
    f = C.c_uint64(0)
    _check(N.lib().bkg_bop(ctx.handle, a.device(ctx), x.shape[1], _dp(x), _dp(y), C.byref(f)))
    if flops is not None:
        flops.multiply_adds_bop += f.value
    return y


def bsolve(gamma: BlockCoefficient, delta: BlockCoefficient,
           ctx: Optional[Context] = None) -> BlockCoefficient:
    """BSOLVE gamma^-1 delta blockwise (kernels.hpp:231-240)."""
    if not gamma.config == delta.config:
        raise DimensionError("bsolve: gamma and delta use different subalgebra configurations")
    cfg = gamma.config
    ctx = ctx or default_context()
    out = BlockCoefficient(cfg)
    bad = C.c_uint64(0)
    g = np.ascontiguousarray(gamma.data)
    d = np.ascontiguousarray(delta.data)
    st = N.lib().bkg_bsolve(ctx.handle, cfg.k, cfg.p, cfg._mode_code, _dp(g), _dp(d),
                            _dp(out.data), C.byref(bad))
    _check(st, block=int(bad.value))
    return out


def column_norms(x, ctx: Optional[Context] = None) -> np.ndarray:
    """Per-column Euclidean norms (block_vector.hpp:59-70)."""
    x = _bv(x)
    ctx = ctx or default_context()
    out = np.empty(x.shape[1])
    _check(N.lib().bkg_column_norms(ctx.handle, x.shape[0], x.shape[1], _dp(x), _dp(out)))
    return out


# --------------------------------------------------------- preconditioner --
IDENTITY = "identity"
JACOBI = "jacobi"
ILU0 = "ilu0"
_PREC = {IDENTITY: 0, JACOBI: 1, ILU0: 2}


class Preconditioner:
    """Column-wise M^-1 (preconditioners.hpp:66-147)."""

    def __init__(self, kind: str, n: int, matrix: Optional[SparseMatrix] = None):
        self._kind, self._n, self.matrix = kind, n, matrix

    @staticmethod
    def identity(n: int) -> "Preconditioner":
        return Preconditioner(IDENTITY, n)

    @staticmethod
    def jacobi(a: SparseMatrix) -> "Preconditioner":
        bad = np.flatnonzero(~(a.diagonal() > 0.0))
        if bad.size:
            r = int(bad[0])
            raise FactorizationError(r, f"jacobi: diagonal entry {r} is not strictly positive")
        return Preconditioner(JACOBI, a.n(), a)

    def kind(self) -> str:
        return self._kind

    def n(self) -> int:
        return self._n

    def apply(self, r, z: Optional[np.ndarray] = None, flops: Optional[FlopCounter] = None,
              ctx: Optional[Context] = None) -> np.ndarray:
        r = _bv(r)
        if r.shape[0] != self._n:
            raise DimensionError(f"preconditioner: expected {self._n} rows, got {r.shape[0]}")
        if z is None or z.shape != r.shape:
            z = np.empty_like(r)
        if self._kind == IDENTITY:  # preconditioners.hpp:81-84 (a copy)
            z[...] = r
            return z
        ctx = ctx or default_context()
        f = C.c_uint64(0)
        _check(N.lib().bkg_precond_apply(ctx.handle, self.matrix.device(ctx), _PREC[self._kind],
                                         r.shape[1], _dp(r), _dp(z), C.byref(f)))
        if flops is not None:
            flops.multiply_adds_precond += f.value
        return z


def _precond_setup(a: SparseMatrix, kind: str, ctx: Optional[Context] = None) -> None:
    ctx = ctx or default_context()
    bad = C.c_int64(-1)
    st = N.lib().bkg_precond_setup(ctx.handle, a.device(ctx), _PREC[kind], C.byref(bad))
    _check(st, row=int(bad.value))


def ilu0_factor(a: SparseMatrix, ctx: Optional[Context] = None) -> Preconditioner:
    """ILU(0) (preconditioners.hpp:153-196), factored on the device now (so a
    zero pivot raises FactorizationError here, as in the reference)."""
    _precond_setup(a, ILU0, ctx)
    return Preconditioner(ILU0, a.n(), a)


# ------------------------------------------------------------------ solver -
@dataclass
class SolveOptions:
    """solver.hpp:21-32."""

    tol: float = 1e-8
    max_iter: int = 0
    record_history: bool = False
    on_iterate: Optional[Callable[[int, np.ndarray, np.ndarray], None]] = None
    # per-kernel-class device seconds into SolveReport.seconds (bkg.h time_kernels)
    time_kernels: bool = False


@dataclass
class BreakdownInfo:
    iteration: int
    block_index: int


@dataclass
class KernelSeconds:
    bdot: float = 0.0
    baxpy: float = 0.0
    bop: float = 0.0
    precond: float = 0.0


@dataclass
class SolveReport:
    """solver.hpp:48-59 (+ loop_seconds: device time of the iteration loop)."""

    iterations: int = 0
    converged: bool = False
    defect_history: List[np.ndarray] = field(default_factory=list)
    flops: FlopCounter = field(default_factory=FlopCounter)
    breakdown: Optional[BreakdownInfo] = None
    final_defect_norms: np.ndarray = field(default_factory=lambda: np.zeros(0))
    seconds: KernelSeconds = field(default_factory=KernelSeconds)
    loop_seconds: float = 0.0


@dataclass
class SolveResult:
    x: np.ndarray
    report: SolveReport


def bcg_solve(a: SparseMatrix, b, *args, ctx: Optional[Context] = None,
              out: Optional[np.ndarray] = None) -> SolveResult:
    """bcg_solve(a, b, [x0,] m, cfg, opts=SolveOptions()) — solver.hpp:106-216.

    ``out`` (optional, (n, k) float64 C-order, e.g. pinned host memory) receives
    X instead of a freshly allocated array."""
    if len(args) and isinstance(args[0], np.ndarray):
        x0, rest = args[0], args[1:]
    else:
        x0, rest = None, args
    m: Preconditioner = rest[0]
    cfg: SubalgebraConfig = rest[1]
    opts: SolveOptions = rest[2] if len(rest) > 2 else SolveOptions()
    b = _bv(b)
    if a.n() != b.shape[0]:
        raise DimensionError(f"bcg_solve: matrix dimension {a.n()} does not match right hand "
                             f"side rows {b.shape[0]}")
    if b.shape[1] != cfg.k:
        raise DimensionError(f"bcg_solve: right hand side has k={b.shape[1]} but configuration "
                             f"expects k={cfg.k}")
    if x0 is not None:
        x0 = _bv(x0)
        if x0.shape != b.shape:
            raise DimensionError("bcg_solve: initial guess shape does not match right hand side")
    if m.n() != a.n():
        raise DimensionError("bcg_solve: preconditioner dimension does not match matrix")
    if not opts.tol > 0.0:
        raise ConfigError("bcg_solve: tol must be positive")
    ctx = ctx or default_context()
    n, k = b.shape
    if out is not None:
        if out.shape != b.shape or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise DimensionError("bcg_solve: out must be a C-contiguous float64 (n x k) array")
        x = out
    else:
        x = np.empty_like(b)
    fin = np.empty(k)
    rep = N.Report()
    so = N.SolveOptions()
    so.tol = float(opts.tol)
    so.max_iter = int(opts.max_iter)
    so.record_history = 1 if opts.record_history else 0
    so.precond = _PREC[m.kind()]
    so.time_kernels = 1 if opts.time_kernels else 0
    cb_holder = None
    errors: List[BaseException] = []
    if opts.on_iterate is not None:
        def _cb(i, xp, rp, nn, kk, user):
            try:
                xv = np.ctypeslib.as_array(xp, shape=(nn, kk)).copy()
                rv = np.ctypeslib.as_array(rp, shape=(nn, kk)).copy()
                opts.on_iterate(int(i), xv, rv)
            except BaseException as e:  # surface after the call returns
                errors.append(e)
        cb_holder = N.ITERATE_FN(_cb)
        so.on_iterate = cb_holder
    x0p = _dp(x0) if x0 is not None else None
    st = N.lib().bkg_solve(ctx.handle, a.device(ctx), cfg.k, cfg.p, cfg._mode_code, _dp(b), x0p,
                           C.byref(so), _dp(x), None, 0, _dp(fin), C.byref(rep))
    _check(st)
    if errors:
        raise errors[0]
    report = SolveReport(
        iterations=int(rep.iterations), converged=bool(rep.converged),
        flops=FlopCounter(int(rep.flops_bdot), int(rep.flops_baxpy), int(rep.flops_bop),
                          int(rep.flops_precond)),
        final_defect_norms=fin,
        seconds=KernelSeconds(rep.seconds_bdot, rep.seconds_baxpy, rep.seconds_bop,
                              rep.seconds_precond),
        loop_seconds=float(rep.loop_seconds))
    if rep.breakdown:
        report.breakdown = BreakdownInfo(int(rep.breakdown_iteration), int(rep.breakdown_block))
    if opts.record_history:  # sized from the rows produced (solver.hpp:146,198)
        rows = int(rep.history_rows)
        hist = np.empty((max(rows, 1), k))
        got = C.c_uint64(0)
        _check(N.lib().bkg_solve_history(ctx.handle, _dp(hist), rows, C.byref(got)))
        report.defect_history = [hist[i].copy() for i in range(min(rows, got.value))]
    return SolveResult(x, report)


# ------------------------------------------------------------ generators ---
POISSON2D_CONST, POISSON2D_LOGUNI, DIFFUSION2D_LOGNORMAL, LAPLACE3D_7PT, STENCIL3D_27PT = range(5)


def stencil(kind: int, nx: int, ny: int, nz: int = 1, seed: int = 0, contrast: float = 2.0,
            validate: bool = False) -> SparseMatrix:
    """Generator kinds of bkg_stencil_fill (problems.hpp:74-124 + DESIGN.md §Inputs)."""
    n = C.c_uint64()
    nnz = C.c_uint64()
    _check(N.lib().bkg_stencil_size(kind, nx, ny, nz, C.byref(n), C.byref(nnz)))
    off = np.empty(n.value + 1, dtype=np.uint64)
    cols = np.empty(nnz.value, dtype=np.uint64)
    vals = np.empty(nnz.value)
    _check(N.lib().bkg_stencil_fill(kind, nx, ny, nz, seed, contrast, _up(off), _up(cols),
                                    _dp(vals)))
    return SparseMatrix(n.value, off, cols, vals, validate=validate)


@dataclass
class PoissonSpec:
    """problems.hpp:51-66."""

    nx: int = 32
    ny: int = 32
    coefficients: str = "constant"
    contrast: float = 2.0
    seed: int = 0

    @staticmethod
    def constant(nx: int, ny: int) -> "PoissonSpec":
        return PoissonSpec(nx, ny, "constant", 0.0, 0)

    @staticmethod
    def heterogeneous(nx: int, ny: int, seed: int, contrast: float = 2.0) -> "PoissonSpec":
        return PoissonSpec(nx, ny, "log_uniform", contrast, seed)


def poisson2d(spec: PoissonSpec) -> SparseMatrix:
    """problems.hpp:74-124."""
    if spec.nx < 2 or spec.ny < 2:
        raise ConfigError("poisson2d: grid must be at least 2 x 2 cells")
    kind = POISSON2D_CONST if spec.coefficients == "constant" else POISSON2D_LOGUNI
    if kind == POISSON2D_LOGUNI and not spec.contrast >= 0.0:
        raise ConfigError("poisson2d: contrast exponent must be non-negative")
    return stencil(kind, spec.nx, spec.ny, 1, spec.seed, spec.contrast, validate=False)


def random_block_rhs(n: int, k: int, seed: int, out: Optional[np.ndarray] = None) -> np.ndarray:
    """problems.hpp:128-134 — U(-1,1), one xorshift64* stream, row-major."""
    b = out if out is not None else np.empty((n, k))
    _check(N.lib().bkg_random_block_rhs(n, k, seed, _dp(b)))
    return b


def normal_block_rhs(n: int, k: int, seed: int, out: Optional[np.ndarray] = None) -> np.ndarray:
    """Frozen N(0,1) block."""
    b = out if out is not None else np.empty((n, k))
    _check(N.lib().bkg_normal_block_rhs(n, k, seed, _dp(b)))
    return b
