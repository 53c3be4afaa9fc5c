"""Fused fast path on irregular CSR structure: variable row lengths, a wide
(hub) row spanning several sliced-ELL chunks, rows without a stored diagonal,
and n not a multiple of any K1 warp tile.  The first K1 launch (sliced-ELL
SpMM + alpha + on-device lambda) and whole solves are checked against the CPU
oracle.  Solves: X within 1e-8 and, where the reference is reorder-stable on
the instance (its own drift under a row reversal <= 1e-9), the literal
north_star bars (history 1e-9 relative per iteration, iterations +-1); on
these random diagonally dominant graphs the reference's own reversal drift is
O(0.1-1) (fast convergence, ill-conditioned block Krylov basis), so there the
iteration count must agree within 5% (DESIGN.md §2 floor protocol)."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_1912_11930_b200 as bk

pytestmark = pytest.mark.gpu

SHAPES = [(8, 8, False), (8, 2, True), (16, 16, False), (16, 4, True), (32, 8, False),
          (32, 1, False), (32, 16, False), (64, 16, False), (64, 4, True), (64, 1, False)]


def irregular(n, seed, hub=60, drop_diag=0):
    """Symmetric, strictly diagonally dominant (SPD) CSR with 0-11 random
    neighbours per row plus a hub row 0 coupled to `hub` rows; `drop_diag`
    rows lose their stored diagonal (then not SPD: first-step tests only)."""
    rng = np.random.default_rng(seed)
    deg = rng.integers(0, 12, size=n)
    r = np.repeat(np.arange(n), deg)
    c = rng.integers(0, n, size=r.size)
    hubs = rng.choice(np.arange(1, n), size=min(hub, n - 1), replace=False)
    r = np.concatenate([r, np.zeros(hubs.size, dtype=np.int64)])
    c = np.concatenate([c, hubs])
    keep = r != c
    r, c = r[keep], c[keep]
    v = -rng.uniform(0.1, 1.0, size=r.size)
    off = sp.coo_matrix((np.concatenate([v, v]), (np.concatenate([r, c]), np.concatenate([c, r]))),
                        shape=(n, n)).tocsr()
    off.sum_duplicates()
    d = np.asarray(abs(off).sum(axis=1)).ravel() + 1.0
    a = (off + sp.diags(d)).tocsr()
    if drop_diag:
        a = a.tolil()
        for i in rng.choice(n, size=drop_diag, replace=False):
            a[i, i] = 0.0
        a = a.tocsr()
        a.eliminate_zeros()
    a.sort_indices()
    return (a.indptr.astype(np.uint64), a.indices.astype(np.uint64), a.data.astype(np.float64))


@pytest.mark.parametrize("k,p,glob", SHAPES)
@pytest.mark.parametrize("n,drop", [(1001, 0), (333, 40)])
def test_first_step_irregular(port, k, p, glob, n, drop):
    csr = irregular(n, seed=n + k + p, drop_diag=drop)
    a = bk.SparseMatrix(n, *csr, validate=False)
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


@pytest.mark.parametrize("k,p,glob", SHAPES)
def test_solve_irregular_meets_parity_bars(port, k, p, glob):
    n = 2053
    csr = irregular(n, seed=5 + k + p)
    a = bk.SparseMatrix(n, *csr)
    b = bk.normal_block_rhs(n, k, 7)
    ctx = bk.Context(0, "fast")
    cfg = bk.SubalgebraConfig(k, p, "global" if glob else "hybrid")
    opts = bk.SolveOptions(tol=1e-8, max_iter=500, record_history=True)
    res = bk.bcg_solve(a, b, bk.Preconditioner.identity(n), cfg, opts, ctx=ctx)
    ref = port.bcg_solve(csr, b, p, glob and p != k, tol=1e-8, max_iter=500,
                         record_history=True)
    r = res.report
    assert r.converged and ref.report.converged
    xr = np.linalg.norm(res.x - ref.x, axis=0) / np.linalg.norm(ref.x, axis=0)
    assert np.max(xr) <= 1e-8, xr
    floor = _reversal_floor(port, csr, b, p, glob and p != k, ref.history)
    h = np.array(r.defect_history)
    if floor <= 1e-9:
        assert abs(r.iterations - ref.report.iterations) <= 1
        assert _drift(h, ref.history) <= 1e-9
    else:
        assert abs(r.iterations - ref.report.iterations) <= max(1, int(0.05 * ref.report.iterations))
    ctx.close()


def _drift(h, ref):
    rows = min(len(h), len(ref))
    return float(np.max(np.abs(h[:rows] - ref[:rows]) / np.abs(ref[:rows])))


def _reversal_floor(port, csr, b, p, glob, hist):
    """The reference's own history drift when the same system is solved with
    rows and columns in reversed order (tests/make_golden.py protocol)."""
    n = len(csr[0]) - 1
    a = sp.csr_matrix((csr[2], csr[1].astype(np.int64), csr[0].astype(np.int64)), shape=(n, n))
    perm = np.arange(n)[::-1]
    ar = a[perm][:, perm].tocsr()
    ar.sort_indices()
    rev = port.bcg_solve((ar.indptr.astype(np.uint64), ar.indices.astype(np.uint64), ar.data),
                         np.ascontiguousarray(b[perm]), p, glob, tol=1e-8, max_iter=500,
                         record_history=True)
    return _drift(rev.history, hist)


@pytest.mark.parametrize("k,p,glob", [(8, 4, False), (16, 16, False), (32, 8, False),
                                      (64, 4, True)])
@pytest.mark.parametrize("hub", [60, 8])
def test_ilu_irregular_exact_bitwise_and_fast_bars(port, k, p, glob, hub):
    """ILU(0) on an irregular pattern: hub = 60 puts more than 16 entries in a
    triangle row (CSR sweeps), hub = 8 keeps every row ELL-sized; the row
    segments of the sync-free sweeps are mostly single rows here (random
    pattern, few previous-row chains).  Exact mode must be bitwise the
    reference; fast mode meets X 1e-8 and the iteration bars."""
    n = 1499
    csr = irregular(n, seed=17 + k + p + hub, hub=hub)
    a = bk.SparseMatrix(n, *csr)
    b = bk.normal_block_rhs(n, k, 7)
    cfg = bk.SubalgebraConfig(k, p, "global" if glob else "hybrid")
    opts = bk.SolveOptions(tol=1e-8, max_iter=300, record_history=True)
    ref = port.bcg_solve(csr, b, p, glob and p != k, tol=1e-8, max_iter=300,
                         record_history=True, precond="ilu0")
    for mode in ("exact", "fast"):
        ctx = bk.Context(0, mode)
        res = bk.bcg_solve(a, b, bk.ilu0_factor(a, ctx), cfg, opts, ctx=ctx)
        r = res.report
        assert r.converged and ref.report.converged
        if mode == "exact":
            assert r.iterations == ref.report.iterations
            assert np.array(r.defect_history).tobytes() == ref.history.tobytes()
            assert res.x.tobytes() == ref.x.tobytes()
        else:
            xr = np.linalg.norm(res.x - ref.x, axis=0) / np.linalg.norm(ref.x, axis=0)
            assert np.max(xr) <= 1e-8, xr
            assert abs(r.iterations - ref.report.iterations) <= max(1, int(0.05 * ref.report.iterations))
        ctx.close()
