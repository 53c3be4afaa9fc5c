"""k1_line (kernels_k1.cuh): K1 over the line variant of the sliced-ELL copy,
which keeps P[r-1], P[r], P[r+1] of a run of consecutive rows in registers and
takes the entries in those columns out of the slots.  The solver picks it per
matrix (api.cu use_line); BKG_K1_LINE=1 forces it here so every shape runs it:
stencils (3-point lines inside 5/7/27-point rows), a tridiagonal matrix (no
slots left at all), irregular CSR with missing diagonals and ragged n, and n
smaller than one super tile.  First K1 launch vs the oracle, then whole fast
solves against the north_star bars."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_1912_11930_b200 as bk
from test_gpu_irregular import irregular, _drift

pytestmark = pytest.mark.gpu

SHAPES = [(8, 8, False), (8, 4, True), (16, 16, False), (16, 4, True), (32, 8, False),
          (32, 1, False), (64, 16, False), (64, 4, True), (64, 1, False), (4, 2, False)]


@pytest.fixture(params=["line", "wide", "stage"])
def k1_choice(request, monkeypatch):
    """Force one K1: k1_line, k1_wide, or k1_stage (TMA-staged blocks)."""
    monkeypatch.setenv("BKG_K1_LINE", "1" if request.param == "line" else "0")
    monkeypatch.setenv("BKG_K1_STAGE", "1" if request.param == "stage" else "0")
    monkeypatch.setenv("BKG_K1_GRID", "0")
    return request.param


def tridiagonal(n, seed):
    rng = np.random.default_rng(seed)
    off = -rng.uniform(0.1, 1.0, size=n - 1)
    a = sp.diags([off, np.full(n, 2.5), off], [-1, 0, 1]).tocsr()
    a.sort_indices()
    return (a.indptr.astype(np.uint64), a.indices.astype(np.uint64), a.data.astype(np.float64))


def _first_step(port, csr, n, k, p, glob):
    a = bk.SparseMatrix(n, *csr)
    b = bk.normal_block_rhs(n, k, 7)
    ctx = bk.Context(0, "fast")
    s = bk.DeviceSolver(a, bk.SubalgebraConfig(k, p, "global" if glob else "hybrid"), ctx)
    s.set_rhs(b)
    q, coef = s.debug_first_step()
    qref = port.bop(csr, b)
    np.testing.assert_allclose(q, qref, rtol=1e-13, atol=1e-12)
    gl = glob and p != k
    alpha = port.bdot(b, qref, p, gl)
    rho = port.bdot(b, b, p, gl)
    lam, bad = port.bsolve(alpha, rho, k, p, gl)
    cs = alpha.size
    np.testing.assert_allclose(coef[cs:], rho.ravel(), rtol=1e-11)
    if bad is None:
        np.testing.assert_allclose(coef[:cs], lam.ravel(), rtol=1e-9, atol=1e-12)
    s.close()
    ctx.close()


def _csr(a):
    return (a.row_offsets(), a.col_indices(), a.values())


@pytest.mark.parametrize("k,p,glob", SHAPES)
@pytest.mark.parametrize("kind,dims", [(3, (33, 17, 9)), (0, (77, 31, 1)), (4, (11, 9, 13)),
                                       (2, (64, 45, 1)), (3, (6, 5, 4))])
def test_line_first_step_stencils(port, k1_choice, k, p, glob, kind, dims):
    a = bk.stencil(kind, *dims, seed=11)
    _first_step(port, _csr(a), a.n(), k, p, glob)


@pytest.mark.parametrize("k,p,glob", SHAPES)
@pytest.mark.parametrize("n,what", [(1001, "irregular"), (333, "drop"), (517, "tridiagonal"),
                                    (1, "tridiagonal")])
def test_line_first_step_irregular(port, k1_choice, k, p, glob, n, what):
    if what == "tridiagonal":
        csr = tridiagonal(n, 3) if n > 1 else (np.array([0, 1], np.uint64),
                                               np.array([0], np.uint64), np.array([2.0]))
    else:
        csr = irregular(n, seed=n + k, drop_diag=40 if what == "drop" else 0)
    _first_step(port, csr, n, k, p, glob)


@pytest.mark.parametrize("k,p,glob", [(32, 8, False), (64, 16, False), (64, 4, True),
                                      (16, 16, False), (8, 8, False)])
def test_line_solve_meets_parity_bars(port, monkeypatch, k, p, glob):
    """3D 7-point stencils are reorder-stable (reversal floor <= 4e-12,
    DESIGN.md §2), so the literal bars apply: history 1e-9 relative per
    iteration, iterations +-1, X 1e-8."""
    monkeypatch.setenv("BKG_K1_LINE", "1")
    monkeypatch.setenv("BKG_K1_STAGE", "0")
    monkeypatch.setenv("BKG_K1_GRID", "0")
    a = bk.stencil(3, 40, 36, 29, seed=11)
    n = a.n()
    b = bk.normal_block_rhs(n, k, 7)
    ctx = bk.Context(0, "fast")
    cfg = bk.SubalgebraConfig(k, p, "global" if glob else "hybrid")
    opts = bk.SolveOptions(tol=1e-8, max_iter=2000, record_history=True)
    res = bk.bcg_solve(a, b, bk.Preconditioner.identity(n), cfg, opts, ctx=ctx)
    ref = port.bcg_solve(_csr(a), b, p, glob and p != k, tol=1e-8, max_iter=2000,
                         record_history=True)
    r = res.report
    assert r.converged and ref.report.converged
    assert abs(r.iterations - ref.report.iterations) <= 1
    assert _drift(np.array(r.defect_history), ref.history) <= 1e-9
    xr = np.linalg.norm(res.x - ref.x, axis=0) / np.linalg.norm(ref.x, axis=0)
    assert np.max(xr) <= 1e-8, xr
    ctx.close()


def test_line_and_wide_agree_on_large_system(monkeypatch):
    """At the C5 kernel table (3D 7-point 96^3, k = 64, p = 16), a
    fixed-iteration solve with the solver's own choice (k1_grid: the matrix
    is a constant-coefficient grid stencil), k1_stage, k1_line and k1_wide:
    the K1s sum a row's products in different orders only."""
    a = bk.stencil(3, 96, 96, 96, seed=11)
    n = a.n()
    b = bk.normal_block_rhs(n, 64, 7)
    cfg = bk.SubalgebraConfig(64, 16, "hybrid")
    opts = bk.SolveOptions(tol=1e-300, max_iter=40, record_history=True)
    out = {}
    kernels = {}
    for v in ("auto", "1", "0", "stage"):
        monkeypatch.delenv("BKG_K1_LINE", raising=False)
        monkeypatch.delenv("BKG_K1_STAGE", raising=False)
        monkeypatch.delenv("BKG_K1_GRID", raising=False)
        if v != "auto":
            monkeypatch.setenv("BKG_K1_GRID", "0")
        if v in ("1", "0"):
            monkeypatch.setenv("BKG_K1_LINE", v)
            monkeypatch.setenv("BKG_K1_STAGE", "0")
        elif v == "stage":
            monkeypatch.setenv("BKG_K1_STAGE", "1")
        ctx = bk.Context(0, "fast")
        res = bk.bcg_solve(a, b, bk.Preconditioner.identity(n), cfg, opts, ctx=ctx)
        out[v] = (res.x, np.array(res.report.defect_history))
        kernels[v] = ctx.last_k1()
        ctx.close()
    auto = kernels.pop("auto")
    assert kernels == {"1": "k1_line", "0": "k1_wide", "stage": "k1_stage"}
    assert auto == "k1_grid"
    for v in ("auto", "0", "stage"):
        assert _drift(out[v][1], out["1"][1]) <= 1e-9
        xr = np.linalg.norm(out[v][0] - out["1"][0], axis=0) / np.linalg.norm(out["1"][0], axis=0)
        assert np.max(xr) <= 1e-9, xr
    monkeypatch.delenv("BKG_K1_LINE", raising=False)
    monkeypatch.delenv("BKG_K1_STAGE", raising=False)
    monkeypatch.delenv("BKG_K1_GRID", raising=False)
    ctx = bk.Context(0, "fast")
    again = bk.bcg_solve(a, b, bk.Preconditioner.identity(n), cfg, opts, ctx=ctx)
    ctx.close()
    assert out["auto"][0].tobytes() == again.x.tobytes()  # deterministic per kernel
