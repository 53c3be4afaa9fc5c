"""The reference's text formats in Python (host side), byte-compatible with
the C++ drop-in ``include/blockkrylov/io.hpp``:

* Matrix Market coordinate (sparse_matrix.hpp:133-205): written "real
  symmetric", lower triangle, 1-based, ``%.17g``; read symmetric (mirrored)
  or general and assembled with ``SparseMatrix.from_triplets``.
* dense block-vector text (block_vector.hpp:72-112): "n k" then n rows of k
  ``%.17g`` values.
Failures raise :class:`IoError`.
"""
from __future__ import annotations

import numpy as np

from .blockkrylov import Error, SparseMatrix


class IoError(Error):
    """errors.hpp IoError."""


def _g17(v: float) -> str:
    return "%.17g" % v


def save_matrix_market(path: str, a: SparseMatrix) -> None:
    rp, cl, vl = a.row_offsets(), a.col_indices(), a.values()
    rows = np.repeat(np.arange(a.n(), dtype=np.uint64), np.diff(rp).astype(np.int64))
    low = cl <= rows
    try:
        with open(path, "w") as f:
            f.write("%%MatrixMarket matrix coordinate real symmetric\n")
            f.write(f"{a.n()} {a.n()} {int(low.sum())}\n")
            f.writelines(f"{r + 1} {c + 1} {_g17(v)}\n"
                         for r, c, v in zip(rows[low].tolist(), cl[low].tolist(), vl[low].tolist()))
    except OSError as e:
        raise IoError(f"cannot open '{path}' for writing") from e


def load_matrix_market(path: str) -> SparseMatrix:
    try:
        with open(path) as f:
            lines = f.read().split("\n")
    except OSError as e:
        raise IoError(f"cannot open '{path}'") from e
    if not lines or not lines[0]:
        raise IoError("matrix market: empty file")
    h = lines[0].split() + [""] * 5
    if h[0] != "%%MatrixMarket" or h[1] != "matrix" or h[2] != "coordinate":
        raise IoError("matrix market: expected '%%MatrixMarket matrix coordinate' header")
    if h[3] != "real":
        raise IoError("matrix market: only real matrices are supported")
    if h[4] not in ("symmetric", "general"):
        raise IoError(f"matrix market: unsupported symmetry '{h[4]}'")
    i = 1
    while i < len(lines) and (not lines[i] or lines[i][0] == "%"):
        i += 1
    try:
        rows, cols, entries = (int(x) for x in lines[i].split()[:3])
    except (IndexError, ValueError):
        raise IoError("matrix market: missing size line") from None
    if rows != cols:
        raise IoError("matrix market: matrix must be square")
    tok = " ".join(lines[i + 1:]).split()
    if len(tok) < 3 * entries:
        raise IoError("matrix market: truncated entry list")
    trip = []
    for e in range(entries):
        try:
            r, c, v = int(tok[3 * e]), int(tok[3 * e + 1]), float(tok[3 * e + 2])
        except ValueError:
            raise IoError("matrix market: truncated entry list") from None
        if r < 1 or c < 1 or r > rows or c > cols:
            raise IoError("matrix market: entry index out of range")
        trip.append((r - 1, c - 1, v))
        if h[4] == "symmetric" and r != c:
            trip.append((c - 1, r - 1, v))
    return SparseMatrix.from_triplets(rows, trip)


def save_block_vector(path: str, x: np.ndarray) -> None:
    x = np.asarray(x, dtype=np.float64)
    try:
        with open(path, "w") as f:
            f.write(f"{x.shape[0]} {x.shape[1]}\n")
            f.writelines(" ".join(_g17(v) for v in row) + "\n" for row in x.tolist())
    except OSError as e:
        raise IoError(f"cannot open '{path}' for writing") from e


def load_block_vector(path: str) -> np.ndarray:
    try:
        with open(path) as f:
            tok = f.read().split()
    except OSError as e:
        raise IoError(f"cannot open '{path}'") from e
    try:
        n, k = int(tok[0]), int(tok[1])
    except (IndexError, ValueError):
        raise IoError("block vector file: missing 'n k' header") from None
    if k == 0:
        raise IoError("block vector file: column count must be positive")
    vals = []
    for t in tok[2:2 + n * k]:
        try:
            vals.append(float(t))
        except ValueError:
            break  # the stream extraction stops here (block_vector.hpp:101-105)
    if len(vals) < n * k:
        raise IoError(f"block vector file: expected {n * k} entries, file ended early")
    return np.array(vals, dtype=np.float64).reshape(n, k)
