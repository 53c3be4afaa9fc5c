"""Preconditioned solves on the GPU (Jacobi, ILU(0)): the reference's own
ILU-based solver and acceptance tests (proj/tests/test_solver.cpp:153-377,
acceptance_test.cpp:70-186,309-325) restated with their original parameters,
plus standalone apply / factorization against the oracle."""
import numpy as np
import pytest

import paper_1912_11930_b200 as bk

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["exact", "fast"])
def ctx(request):
    c = bk.Context(0, request.param)
    yield c
    c.close()


def dense(a):
    n = a.n()
    d = np.zeros((n, n))
    rp, cl, vl = a.row_offsets(), a.col_indices(), a.values()
    for r in range(n):
        d[r, cl[rp[r]:rp[r + 1]]] = vl[rp[r]:rp[r + 1]]
    return d


@pytest.mark.parametrize("kind", ["jacobi", "ilu0"])
@pytest.mark.parametrize("k", [1, 3, 8])
def test_apply_bitwise_oracle(ctx, port, kind, k):
    a = bk.poisson2d(bk.PoissonSpec.heterogeneous(13, 11, 5))
    r = bk.random_block_rhs(a.n(), k, 17)
    m = bk.ilu0_factor(a, ctx) if kind == "ilu0" else bk.Preconditioner.jacobi(a)
    f = bk.FlopCounter()
    z = m.apply(r, flops=f, ctx=ctx)
    csr = (a.row_offsets(), a.col_indices(), a.values())
    inv = np.zeros(a.n())
    lu = np.zeros(a.nnz())
    import ctypes as C
    from oracle import PRECOND
    lib = port.lib
    lib.orc_precond_setup.argtypes = [C.c_int, C.c_size_t] + [np.ctypeslib.ndpointer(np.uint64)] * 2 + \
        [np.ctypeslib.ndpointer(np.float64)] * 3
    lib.orc_precond_setup.restype = C.c_int64
    assert lib.orc_precond_setup(PRECOND[kind], a.n(), *csr, inv, lu) == 0
    lib.orc_precond_apply.argtypes = [C.c_int, C.c_size_t] + [np.ctypeslib.ndpointer(np.uint64)] * 2 + \
        [np.ctypeslib.ndpointer(np.float64)] * 2 + [C.c_size_t] + \
        [np.ctypeslib.ndpointer(np.float64)] * 2 + [C.POINTER(C.c_uint64)]
    want = np.empty_like(r)
    fl = C.c_uint64(0)
    lib.orc_precond_apply(PRECOND[kind], a.n(), csr[0], csr[1], inv, lu, k, r, want, C.byref(fl))
    assert z.tobytes() == want.tobytes()
    assert f.multiply_adds_precond == fl.value


def test_ilu_zero_pivot_raises_factorization_error(ctx):
    # diag(1, 0, 1) pattern: zero pivot in row 1 (preconditioners.hpp:190-191)
    a = bk.SparseMatrix.from_triplets(3, [(0, 0, 1.0), (1, 1, 0.0), (2, 2, 1.0)])
    with pytest.raises(bk.FactorizationError) as e:
        bk.ilu0_factor(a, ctx)
    assert e.value.row == 1


def test_ilu_flop_totals_follow_iteration_count(ctx):
    # test_solver.cpp:358-377
    a = bk.poisson2d(bk.PoissonSpec.heterogeneous(8, 8, 61))
    n, k, p, z = 64, 4, 2, a.nnz()
    b = bk.random_block_rhs(n, k, 62)
    res = bk.bcg_solve(a, b, bk.ilu0_factor(a, ctx), bk.SubalgebraConfig(k, p), ctx=ctx)
    i = res.report.iterations
    assert res.report.converged and i >= 1
    f = res.report.flops
    assert f.multiply_adds_bdot == 3 * i * 2 * n * p * p * (k // p)
    assert f.multiply_adds_baxpy == 3 * i * 2 * n * p * p * (k // p)
    assert f.multiply_adds_bop == i * 2 * k * z
    assert f.multiply_adds_precond == (i + 1) * (2 * k * (z - n) + n * k)


def test_acceptance_oracle_correctness_with_ilu(ctx):
    # acceptance_test.cpp:70-99: 32x32 instance, k = 8, ILU, every hybrid width
    a = bk.poisson2d(bk.PoissonSpec.heterogeneous(32, 32, 7))
    b = bk.random_block_rhs(1024, 8, 7)
    xs = np.linalg.solve(dense(a), b)
    m = bk.ilu0_factor(a, ctx)
    iters = {}
    for p in (1, 2, 4, 8):
        res = bk.bcg_solve(a, b, m, bk.SubalgebraConfig(8, p), bk.SolveOptions(tol=1e-8), ctx=ctx)
        assert res.report.converged
        err = np.linalg.norm(res.x - xs, axis=0) / np.linalg.norm(xs, axis=0)
        assert np.all(err <= 1e-6)
        iters[p] = res.report.iterations
    # acceptance_test.cpp:309-325: classical needs no more iterations than parallel
    assert iters[8] <= iters[1]


def _iterates(a, b, m, cfg, iters, ctx):
    out = []
    opts = bk.SolveOptions(tol=1e-30, max_iter=iters, on_iterate=lambda i, x, r: out.append(x))
    bk.bcg_solve(a, b, m, cfg, opts, ctx=ctx)
    return out


def test_hybrid_with_ilu_splits_into_classical_runs(ctx):
    # test_solver.cpp:194-231 (original parameters, ILU)
    a = bk.poisson2d(bk.PoissonSpec.heterogeneous(16, 16, 7))
    b = bk.random_block_rhs(256, 8, 9)
    m = bk.ilu0_factor(a, ctx)
    hy = _iterates(a, b, m, bk.SubalgebraConfig(8, 4), 20, ctx)
    for g in range(2):
        cl = _iterates(a, b[:, 4 * g:4 * g + 4].copy(), m, bk.SubalgebraConfig.classical(4), 20, ctx)
        for i in range(len(hy)):
            assert np.max(np.abs(hy[i][:, 4 * g:4 * g + 4] - cl[i])) <= 1e-12


def test_global_with_ilu_equals_stacked_classical(ctx):
    # test_solver.cpp:236-273 (original parameters, ILU on both systems)
    a = bk.poisson2d(bk.PoissonSpec.heterogeneous(16, 16, 7))
    n, k, p, q = 256, 8, 4, 2
    b = bk.random_block_rhs(n, k, 10)
    gl = _iterates(a, b, bk.ilu0_factor(a, ctx), bk.SubalgebraConfig(k, p, "global"), 20, ctx)
    rp, cl, vl = a.row_offsets(), a.col_indices(), a.values()
    trip = [(c * n + r, c * n + int(cl[i]), vl[i]) for c in range(q) for r in range(n)
            for i in range(rp[r], rp[r + 1])]
    ast = bk.SparseMatrix.from_triplets(q * n, trip)
    bst = np.vstack([b[:, g * p:(g + 1) * p] for g in range(q)])
    st = _iterates(ast, bst, bk.ilu0_factor(ast, ctx), bk.SubalgebraConfig.classical(p), 20, ctx)
    for i in range(len(gl)):
        d = max(np.max(np.abs(gl[i][:, g * p:(g + 1) * p] - st[i][g * n:(g + 1) * n]))
                for g in range(q))
        assert d <= 1e-10


def test_parallel_with_ilu_matches_columnwise_pcg(ctx):
    # test_solver.cpp:153-190: p = 1 with ILU == scalar PCG per column
    a = bk.poisson2d(bk.PoissonSpec.heterogeneous(16, 16, 7))
    n, k, iters = 256, 4, 15
    b = bk.random_block_rhs(n, k, 8)
    m = bk.ilu0_factor(a, ctx)
    blk = _iterates(a, b, m, bk.SubalgebraConfig.parallel(k), iters, ctx)
    A = dense(a)

    def prec(v):
        return m.apply(v.reshape(n, 1).copy(), ctx=ctx).ravel()

    for c in range(k):
        x = np.zeros(n)
        r = b[:, c].copy()
        p = prec(r)
        its = [x.copy()]
        for _ in range(iters):
            qv = A @ p
            alpha, rho_prev = p @ qv, p @ r
            lam = rho_prev / alpha
            x = x + lam * p
            r = r - lam * qv
            z = prec(r)
            p = z + ((z @ r) / rho_prev) * p
            its.append(x.copy())
        for i in range(iters + 1):
            np.testing.assert_allclose(blk[i][:, c], its[i], atol=1e-12 * (1 + np.abs(its[i]).max()))


def test_energy_error_monotone_with_ilu(ctx):
    # test_solver.cpp:275-302
    a = bk.poisson2d(bk.PoissonSpec.heterogeneous(8, 8, 21))
    b = bk.random_block_rhs(64, 4, 22)
    A = dense(a)
    xs = np.linalg.solve(A, b)
    energy = []
    opts = bk.SolveOptions(tol=1e-10, on_iterate=lambda i, x, r: energy.append(
        np.sqrt(np.maximum(np.einsum("ij,ij->j", xs - x, A @ (xs - x)), 0.0))))
    bk.bcg_solve(a, b, bk.ilu0_factor(a, ctx), bk.SubalgebraConfig.classical(4), opts, ctx=ctx)
    e = np.array(energy)
    assert np.all(e[1:] <= e[:-1] * (1 + 1e-10) + 1e-14)


# ------------------------------------------- Jacobi in the fused fast loop --
def test_jacobi_flop_totals_follow_iteration_count(ctx):
    # test_solver.cpp:358-377 with Jacobi: n*k multiplies per apply
    a = bk.poisson2d(bk.PoissonSpec.heterogeneous(8, 8, 61))
    n, k, p, z = 64, 4, 2, a.nnz()
    b = bk.random_block_rhs(n, k, 62)
    res = bk.bcg_solve(a, b, bk.Preconditioner.jacobi(a), bk.SubalgebraConfig(k, p), ctx=ctx)
    i = res.report.iterations
    assert res.report.converged and i >= 1
    f = res.report.flops
    assert f.multiply_adds_bdot == 3 * i * 2 * n * p * p * (k // p)
    assert f.multiply_adds_bop == i * 2 * k * z
    assert f.multiply_adds_precond == (i + 1) * n * k


@pytest.mark.parametrize("k", [4, 8, 16])
def test_parallel_with_jacobi_matches_columnwise_pcg(ctx, k):
    # test_solver.cpp:153-190 with M = D: p = 1 block CG == scalar PCG per column
    a = bk.poisson2d(bk.PoissonSpec.heterogeneous(16, 16, 7))
    n, iters = 256, 15
    b = bk.random_block_rhs(n, k, 8)
    m = bk.Preconditioner.jacobi(a)
    blk = _iterates(a, b, m, bk.SubalgebraConfig.parallel(k), iters, ctx)
    A = dense(a)
    dinv = 1.0 / np.diag(A)
    for c in range(k):
        x = np.zeros(n)
        r = b[:, c].copy()
        p = dinv * r
        its = [x.copy()]
        for _ in range(iters):
            qv = A @ p
            alpha, rho_prev = p @ qv, p @ r
            lam = rho_prev / alpha
            x = x + lam * p
            r = r - lam * qv
            z = dinv * r
            p = z + ((z @ r) / rho_prev) * p
            its.append(x.copy())
        for i in range(iters + 1):
            np.testing.assert_allclose(blk[i][:, c], its[i], atol=1e-12 * (1 + np.abs(its[i]).max()))


@pytest.mark.parametrize("k,p,mode", [(16, 8, "hybrid"), (32, 16, "hybrid"), (8, 4, "global"),
                                      (16, 4, "hybrid"), (8, 1, "hybrid")])
def test_fused_jacobi_matches_reference_order(k, p, mode):
    # 3D 7-point with log-uniform coefficients (reorder-stable: floor ~1e-12):
    # the fused loop (K2/K3 scale by D^-1) against the exact-order kernels,
    # which are bit-identical to the reference (c2_16_jacobi fixture).
    a = bk.stencil(3, 14, 13, 12, seed=5)
    b = bk.normal_block_rhs(a.n(), k, 7)
    m = bk.Preconditioner.jacobi(a)
    cfg = bk.SubalgebraConfig(k, p, mode)
    opts = bk.SolveOptions(tol=1e-10, record_history=True)
    out = {}
    for mode_name in ("exact", "fast"):
        c = bk.Context(0, mode_name)
        out[mode_name] = bk.bcg_solve(a, b, m, cfg, opts, ctx=c)
        c.close()
    e, f = out["exact"], out["fast"]
    assert e.report.converged and f.report.converged
    assert abs(e.report.iterations - f.report.iterations) <= 1
    he, hf = np.array(e.report.defect_history), np.array(f.report.defect_history)
    rows = min(len(he), len(hf))
    assert np.max(np.abs(hf[:rows] - he[:rows]) / np.abs(he[:rows])) <= 1e-9
    xs = np.linalg.norm(f.x - e.x, axis=0) / np.linalg.norm(e.x, axis=0)
    assert xs.max() <= 1e-8
    assert f.report.flops.multiply_adds_precond == e.report.flops.multiply_adds_precond
