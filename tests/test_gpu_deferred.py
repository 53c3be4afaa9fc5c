"""Deferred X update in the fused fast loop (K3 skip / flush launches,
DESIGN.md §4): the solve must return the reference's X whatever the parity of
the iteration it stops at -- max_iter, convergence, or a breakdown that hits a
flush iteration with an update still pending.  Fast results are checked
against exact mode (bit-identical to the reference) on the same inputs."""
import numpy as np
import pytest

import paper_1912_11930_b200 as bk

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctxs():
    e, f = bk.Context(0, "exact"), bk.Context(0, "fast")
    yield e, f
    f.close()
    e.close()


def _solve(ctx, a, b, m, cfg, opts):
    return bk.bcg_solve(a, b, m, cfg, opts, ctx=ctx)


@pytest.mark.parametrize("k,p,mode", [(8, 8, "hybrid"), (32, 8, "hybrid"), (16, 4, "global"),
                                      (64, 1, "hybrid"), (64, 16, "hybrid")])
@pytest.mark.parametrize("precond", ["identity", "jacobi", "ilu0"])
def test_fixed_iteration_counts_both_parities(ctxs, k, p, mode, precond):
    ex, fa = ctxs
    a = bk.stencil(3, 12, 10, 9, seed=11)
    n = a.n()
    b = bk.normal_block_rhs(n, k, 7)
    cfg = bk.SubalgebraConfig(k, p, mode)
    for it in range(1, 7):
        opts = bk.SolveOptions(tol=1e-300, max_iter=it)
        out = []
        for c in (ex, fa):
            m = {"identity": lambda: bk.Preconditioner.identity(n),
                 "jacobi": lambda: bk.Preconditioner.jacobi(a),
                 "ilu0": lambda: bk.ilu0_factor(a, c)}[precond]()
            out.append(_solve(c, a, b, m, cfg, opts))
        re, rf = out
        assert rf.report.iterations == re.report.iterations == it
        xr = np.linalg.norm(rf.x - re.x, axis=0) / np.linalg.norm(re.x, axis=0)
        assert np.max(xr) <= 1e-10, (it, xr.max())


def test_breakdown_in_flush_iteration_applies_pending_update(ctxs):
    """Column 0 is an eigenvector: its residual is exactly zero after
    iteration 1, so iteration 2's alpha block (p = 1) is singular and the
    lambda solve breaks down in a flush iteration; X must be X^1."""
    ex, fa = ctxs
    n = 257
    d = 1.0 + np.arange(n) / n
    d[3] = 2.0  # exact: 2 * (1 / 2) == 1, so the column-0 residual is exactly 0
    a = bk.SparseMatrix.from_triplets(n, [(i, i, d[i]) for i in range(n)])
    b = bk.random_block_rhs(n, 4, 5)
    b[:, 0] = 0.0
    b[3, 0] = 1.0
    cfg = bk.SubalgebraConfig(4, 1, "hybrid")
    opts = bk.SolveOptions(tol=1e-300, max_iter=50)
    re = _solve(ex, a, b, bk.Preconditioner.identity(n), cfg, opts)
    rf = _solve(fa, a, b, bk.Preconditioner.identity(n), cfg, opts)
    assert re.report.breakdown is not None
    assert (re.report.breakdown.iteration, re.report.breakdown.block_index) == (2, 0)
    assert rf.report.breakdown is not None
    assert (rf.report.breakdown.iteration, rf.report.breakdown.block_index) == (2, 0)
    assert rf.report.iterations == re.report.iterations == 1
    np.testing.assert_allclose(rf.x, re.x, rtol=1e-13, atol=1e-15)
    assert rf.x[3, 0] == 1.0 / d[3]
