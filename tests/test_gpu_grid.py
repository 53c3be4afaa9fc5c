"""k1_grid (kernels_grid.cuh): K1 for matrices that are exactly a 2-D 5/9-point
or 3-D 7/27-point constant-coefficient grid stencil, applied from TMA-tiled operand
planes (cp.async.bulk.tensor.4d, zero-filled halos) instead of the CSR stream.
The structure is verified entry by entry on device (grid.cu); anything else
keeps the CSR kernels.  BKG_K1_GRID=1 forces it here at every size: first K1
launch vs the oracle (partial tiles, grids smaller than a tile, every slice
count), detection negatives, whole fast solves against the north_star bars."""
import numpy as np
import pytest

import paper_1912_11930_b200 as bk
from test_gpu_irregular import irregular, _drift

pytestmark = pytest.mark.gpu

SHAPES = [(16, 16, False), (16, 4, False), (16, 4, True), (16, 1, False), (32, 8, False),
          (32, 16, False), (32, 2, True), (64, 16, False), (64, 4, True), (64, 1, False),
          (64, 8, False), (128, 16, False), (128, 4, True)]


@pytest.fixture
def grid_on(monkeypatch):
    monkeypatch.setenv("BKG_K1_GRID", "1")
    monkeypatch.setenv("BKG_RESIDENT", "0")  # small systems: not the latency kernel
    monkeypatch.delenv("BKG_K1_LINE", raising=False)
    monkeypatch.delenv("BKG_K1_STAGE", raising=False)


def _csr(a):
    return (a.row_offsets(), a.col_indices(), a.values())


def _first_step(port, csr, n, k, p, glob, expect_grid):
    a = bk.SparseMatrix(n, *csr)
    b = bk.normal_block_rhs(n, k, 7)
    ctx = bk.Context(0, "fast")
    s = bk.DeviceSolver(a, bk.SubalgebraConfig(k, p, "global" if glob else "hybrid"), ctx)
    s.set_rhs(b)
    q, coef = s.debug_first_step()
    assert (s.k1() == "k1_grid") == expect_grid, s.k1()
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


@pytest.mark.parametrize("k,p,glob", SHAPES)
@pytest.mark.parametrize("kind,dims", [(3, (33, 17, 9)), (4, (11, 19, 13)), (3, (16, 16, 16)),
                                       (4, (32, 16, 5)), (3, (6, 5, 4)), (4, (5, 4, 6)),
                                       (3, (47, 35, 3)), (0, (40, 30, 1)), (0, (77, 31, 1)),
                                       (0, (16, 16, 1))])
def test_grid_first_step(port, grid_on, k, p, glob, kind, dims):
    a = bk.stencil(kind, *dims, seed=11)
    _first_step(port, _csr(a), a.n(), k, p, glob, True)


@pytest.mark.parametrize("zchunk", ["1", "2", "3", "5", "100"])
def test_grid_first_step_z_chunks(port, grid_on, monkeypatch, zchunk):
    """Every z-chunk length: items read their two extra planes and emit each row once."""
    monkeypatch.setenv("BKG_GRID_ZCHUNK", zchunk)
    a = bk.stencil(3, 20, 18, 11, seed=11)
    _first_step(port, _csr(a), a.n(), 32, 8, False, True)
    a = bk.stencil(4, 20, 18, 11, seed=11)
    _first_step(port, _csr(a), a.n(), 16, 16, False, True)


@pytest.mark.parametrize("ns", ["2", "3", "4"])
def test_grid_first_step_ring_depths(port, grid_on, monkeypatch, ns):
    monkeypatch.setenv("BKG_GRID_NS", ns)
    a = bk.stencil(3, 35, 33, 12, seed=11)
    _first_step(port, _csr(a), a.n(), 64, 16, False, True)


def test_grid_variable_coefficients_and_rejects(port, grid_on, monkeypatch):
    """Variable coefficients on a 5 / 7-point star run k1_grid from the DIA
    tiles (2-D heterogeneous Poisson, the C3 lognormal field, a 7-point stencil
    with one value changed or one entry pair removed); an odd nx (TMA stride),
    BKG_GRID_VAR=0 and irregular patterns keep the CSR kernels.  All correct."""
    monkeypatch.setenv("BKG_GRID_VAR", "1")
    for kind, dims in [(1, (32, 32, 1)), (2, (32, 24, 1)), (2, (70, 33, 1))]:
        a = bk.stencil(kind, *dims, seed=11)
        for k, p, glob in [(16, 4, False), (64, 1, False), (64, 4, True), (32, 8, False)]:
            _first_step(port, _csr(a), a.n(), k, p, glob, True)
    a = bk.stencil(1, 33, 20, 1, seed=11)  # odd nx
    _first_step(port, _csr(a), a.n(), 16, 4, False, False)
    _first_step(port, irregular(1001, seed=5), 1001, 16, 4, False, False)
    a = bk.stencil(3, 12, 11, 10, seed=11)
    rp, ci, v = (np.array(x) for x in _csr(a))
    n = a.n()
    v2 = v.copy()
    v2[int(rp[n // 3]) + 1] *= 1.0 + 2.0 ** -50  # one coefficient off by a few ulp
    _first_step(port, (rp, ci, v2), n, 16, 4, False, True)
    _first_step(port, (rp, ci, v2), n, 64, 16, False, True)
    # remove one off-diagonal entry and its symmetric counterpart
    row = n // 2 + 3
    e = int(rp[row])
    if ci[e] == row:
        e += 1
    col = int(ci[e])
    e2 = int(rp[col]) + int(np.nonzero(ci[int(rp[col]):int(rp[col + 1])] == row)[0][0])
    keep = np.ones(len(ci), bool)
    keep[[e, e2]] = False
    cnt = np.diff(rp.astype(np.int64))
    cnt[row] -= 1
    cnt[col] -= 1
    rp3 = np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint64)
    _first_step(port, (rp3, ci[keep], v[keep]), n, 16, 4, False, True)
    monkeypatch.delenv("BKG_GRID_VAR")  # on by default, 2-D and 3-D
    _first_step(port, (rp, ci, v2), n, 16, 4, False, True)
    a2 = bk.stencil(2, 32, 24, 1, seed=11)
    _first_step(port, _csr(a2), a2.n(), 16, 4, False, True)
    monkeypatch.setenv("BKG_GRID_VAR", "0")
    _first_step(port, _csr(a2), a2.n(), 16, 4, False, False)
    _first_step(port, (rp, ci, v2), n, 16, 4, False, False)
    monkeypatch.delenv("BKG_GRID_VAR")
    # a small 27-point grid is accepted (constant path)
    a4 = bk.stencil(4, 9, 8, 7, seed=11)
    _first_step(port, _csr(a4), a4.n(), 16, 4, False, True)


@pytest.mark.parametrize("k,p,glob", [(64, 1, False), (64, 4, True), (16, 16, False)])
def test_grid_variable_solve_agrees_with_csr_kernels(grid_on, monkeypatch, k, p, glob):
    """C3's lognormal diffusion at reduced size: whole fast solves with the
    variable-coefficient k1_grid and with k1_wide.  The field is reorder-chaotic
    (DESIGN.md §2 floor), so the bars are X 1e-8 and iterations within 5%."""
    monkeypatch.setenv("BKG_GRID_VAR", "1")
    a = bk.stencil(2, 96, 80, 1, seed=11)
    n = a.n()
    b = bk.random_block_rhs(n, k, 7)
    cfg = bk.SubalgebraConfig(k, p, "global" if glob else "hybrid")
    opts = bk.SolveOptions(tol=1e-10, max_iter=20000)
    out = {}
    for v in ("1", "0"):
        monkeypatch.setenv("BKG_K1_GRID", v)
        ctx = bk.Context(0, "fast")
        res = bk.bcg_solve(a, b, bk.Preconditioner.identity(n), cfg, opts, ctx=ctx)
        assert ctx.last_k1() == ("k1_grid" if v == "1" else "k1_wide")
        assert res.report.converged
        out[v] = (res.x, res.report.iterations)
        ctx.close()
    xr = np.linalg.norm(out["1"][0] - out["0"][0], axis=0) / np.linalg.norm(out["0"][0], axis=0)
    assert np.max(xr) <= 1e-8, xr
    assert abs(out["1"][1] - out["0"][1]) <= max(1, int(0.05 * out["0"][1]))


@pytest.mark.parametrize("kind,k,p,glob", [(3, 32, 8, False), (3, 64, 16, False), (3, 64, 4, True),
                                            (4, 16, 16, False), (4, 16, 4, False),
                                            (4, 16, 4, True), (3, 64, 1, False)])
def test_grid_solve_meets_parity_bars(port, grid_on, kind, k, p, glob):
    """Whole fast solves with k1_grid against the reference port: history 1e-9
    relative per iteration, iterations +-1, X 1e-8 (north_star)."""
    dims = (40, 36, 29) if kind == 3 else (24, 22, 20)
    a = bk.stencil(kind, *dims, seed=11)
    n = a.n()
    b = bk.normal_block_rhs(n, k, 7)
    ctx = bk.Context(0, "fast")
    cfg = bk.SubalgebraConfig(k, p, "global" if glob else "hybrid")
    opts = bk.SolveOptions(tol=1e-8, max_iter=2000, record_history=True)
    res = bk.bcg_solve(a, b, bk.Preconditioner.identity(n), cfg, opts, ctx=ctx)
    assert ctx.last_k1() == "k1_grid"
    ref = port.bcg_solve(_csr(a), b, p, glob and p != k, tol=1e-8, max_iter=2000,
                         record_history=True)
    r = res.report
    assert r.converged and ref.report.converged
    assert abs(r.iterations - ref.report.iterations) <= 1
    assert _drift(np.array(r.defect_history), ref.history) <= 1e-9
    xr = np.linalg.norm(res.x - ref.x, axis=0) / np.linalg.norm(ref.x, axis=0)
    assert np.max(xr) <= 1e-8, xr
    ctx.close()


@pytest.mark.parametrize("kind,dims,k,p", [(3, (96, 96, 96), 64, 16), (4, (64, 64, 48), 16, 16),
                                            (3, (80, 72, 64), 32, 8)])
def test_grid_and_wide_agree_on_large_system(monkeypatch, kind, dims, k, p):
    """Fixed-iteration solves with k1_grid and the CSR k1_wide on the bench
    kernel tables: same histories to 1e-9, deterministic run to run."""
    a = bk.stencil(kind, *dims, seed=11)
    n = a.n()
    b = bk.normal_block_rhs(n, k, 7)
    cfg = bk.SubalgebraConfig(k, p, "hybrid")
    opts = bk.SolveOptions(tol=1e-300, max_iter=40, record_history=True)
    out = {}
    for v in ("grid", "wide", "grid2"):
        monkeypatch.setenv("BKG_K1_GRID", "0" if v == "wide" else "1")
        monkeypatch.setenv("BKG_K1_LINE", "0")
        monkeypatch.setenv("BKG_K1_STAGE", "0")
        ctx = bk.Context(0, "fast")
        res = bk.bcg_solve(a, b, bk.Preconditioner.identity(n), cfg, opts, ctx=ctx)
        assert ctx.last_k1() == ("k1_wide" if v == "wide" else "k1_grid")
        out[v] = (res.x, np.array(res.report.defect_history))
        ctx.close()
    assert _drift(out["grid"][1], out["wide"][1]) <= 1e-9
    xr = np.linalg.norm(out["grid"][0] - out["wide"][0], axis=0) / np.linalg.norm(out["wide"][0],
                                                                                  axis=0)
    assert np.max(xr) <= 1e-9, xr
    assert out["grid"][0].tobytes() == out["grid2"][0].tobytes()


@pytest.mark.parametrize("k,p", [(16, 4), (64, 16), (32, 8)])
def test_grid2_solve_agrees_with_csr_kernels(monkeypatch, k, p):
    """2-D constant 5-point Poisson through k1_grid2 (128-point line tiles
    marching in y, kernels_grid2.cuh) and through the CSR kernels: fixed
    iteration count, X 1e-8, history within 5e-9 (the reference's own
    reordering floor on 2-D Poisson is 6.6e-10)."""
    a = bk.stencil(0, 300, 257, 1, seed=11)
    n = a.n()
    b = bk.normal_block_rhs(n, k, 7)
    cfg = bk.SubalgebraConfig(k, p, "hybrid")
    opts = bk.SolveOptions(tol=1e-300, max_iter=60, record_history=True)
    out = {}
    for v in ("1", "0"):
        monkeypatch.setenv("BKG_K1_GRID", v)
        monkeypatch.setenv("BKG_K1_LINE", "0")
        monkeypatch.setenv("BKG_K1_STAGE", "0")
        ctx = bk.Context(0, "fast")
        res = bk.bcg_solve(a, b, bk.Preconditioner.identity(n), cfg, opts, ctx=ctx)
        assert ctx.last_k1() == ("k1_grid" if v == "1" else "k1_wide")
        out[v] = (res.x, np.array(res.report.defect_history))
        ctx.close()
    assert _drift(out["1"][1], out["0"][1]) <= 5e-9
    xr = np.linalg.norm(out["1"][0] - out["0"][0], axis=0) / np.linalg.norm(out["0"][0], axis=0)
    assert np.max(xr) <= 1e-8, xr
