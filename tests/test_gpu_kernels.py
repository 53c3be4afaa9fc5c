"""GPU kernel parity: BDOT / BAXPY / BOP / BSOLVE / column norms through the
C ABI against the CPU oracle and against the reference's own kernel tests
(proj/tests/test_kernels.cpp, restated).  Exact mode must be bit-identical to
the oracle; fast mode within the tolerances the reference tests use."""
import numpy as np
import pytest

import paper_1912_11930_b200 as bk
from cases import POISSON2D_CONST, POISSON2D_LOGUNI

pytestmark = pytest.mark.gpu

MODES = ["exact", "fast"]


@pytest.fixture(scope="module", params=MODES)
def ctx(request):
    c = bk.Context(0, request.param)
    yield c
    c.close()


@pytest.fixture(scope="module")
def exact():
    c = bk.Context(0, "exact")
    yield c
    c.close()


@pytest.fixture(scope="module")
def fast():
    c = bk.Context(0, "fast")
    yield c
    c.close()


def seeded(n, k, seed):
    return bk.random_block_rhs(n, k, seed)


def unit_block(n, k, port):
    # entries uniform(0,1) from Xorshift64Star(99) (test_kernels.cpp:17-23)
    return ((port.rng_symmetric(99, n * k) + 1.0) / 2.0).reshape(n, k)


def cfg(k, p, glob=False):
    return bk.SubalgebraConfig(k, p, "global" if glob else "hybrid")


# ---------------------------------------------------------------- BDOT ---
def test_bdot_orthonormal_columns_give_identity(ctx):
    x = np.zeros((6, 4))
    for c in range(4):
        x[c, c] = 1.0
    for p in (1, 2, 4):
        g = bk.bdot(x, x, cfg(4, p), ctx=ctx)
        for b in range(g.block_count()):
            np.testing.assert_array_equal(g.block(b), np.eye(p))


def test_bdot_hybrid_and_global_match_dense(ctx):
    x = seeded(4, 4, 7)
    xtx = x.T @ x
    g = bk.bdot(x, x, cfg(4, 2), ctx=ctx)
    for b in range(2):
        np.testing.assert_allclose(g.block(b), xtx[2 * b:2 * b + 2, 2 * b:2 * b + 2], atol=1e-14)
    g = bk.bdot(x, x, cfg(4, 2, True), ctx=ctx)
    np.testing.assert_allclose(g.block(0), xtx[:2, :2] + xtx[2:, 2:], atol=1e-13)


def test_bdot_transpose_symmetry(ctx):
    x, y = seeded(7, 8, 3), seeded(7, 8, 4)
    for glob in (False, True):
        for p in (1, 2, 4, 8):
            xy = bk.bdot(x, y, cfg(8, p, glob), ctx=ctx)
            yx = bk.bdot(y, x, cfg(8, p, glob), ctx=ctx)
            np.testing.assert_allclose(xy.data, np.transpose(yx.data, (0, 2, 1)), atol=1e-14)


def test_bdot_embedding_restriction(ctx):
    for p1, p2, k in ((1, 2, 4), (2, 4, 8)):
        x, y = seeded(9, k, 5), seeded(9, k, 6)
        fine = bk.bdot(x, y, cfg(k, p1), ctx=ctx)
        coarse = bk.bdot(x, y, cfg(k, p2), ctx=ctx)
        per = p2 // p1
        for b in range(k // p1):
            cb, off = b // per, (b % per) * p1
            sub = coarse.block(cb)[off:off + p1, off:off + p1]
            if ctx.numerics == "exact":  # same per-entry order: exact (test_kernels.cpp:108-129)
                np.testing.assert_array_equal(fine.block(b), sub)
            else:
                np.testing.assert_allclose(fine.block(b), sub, atol=1e-14)


def test_bdot_classical_coincidence(ctx):
    x, y = seeded(6, 4, 11), seeded(6, 4, 12)
    hy = bk.bdot(x, y, cfg(4, 4), ctx=ctx)
    gl = bk.bdot(x, y, cfg(4, 4, True), ctx=ctx)
    np.testing.assert_array_equal(hy.block(0), gl.block(0))


def test_bdot_psd(ctx):
    x = seeded(10, 8, 21)
    for glob in (False, True):
        g = bk.bdot(x, x, cfg(8, 4, glob), ctx=ctx)
        for b in range(g.block_count()):
            s = 0.5 * (g.block(b) + g.block(b).T)
            assert np.linalg.eigvalsh(s).min() >= -1e-12


@pytest.mark.parametrize("n,k,p,glob", [
    (7, 8, 1, False), (7, 8, 2, True), (33, 3, 1, False), (33, 6, 3, True), (5, 9, 3, False),
    (1000, 8, 8, False), (4099, 16, 4, True), (4099, 16, 16, False), (3001, 32, 8, False),
    (3001, 64, 1, False), (3001, 64, 4, True), (2049, 64, 16, False), (515, 2, 2, False)])
def test_bdot_exact_is_bitwise_oracle(exact, port, n, k, p, glob):
    x, y = seeded(n, k, 101), seeded(n, k, 102)
    got = bk.bdot(x, y, cfg(k, p, glob), ctx=exact).data
    want = port.bdot(x, y, p, glob and p != k)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("n,k,p,glob", [
    (100003, 8, 8, False), (100003, 16, 4, True), (100003, 16, 16, False),
    (50021, 32, 8, False), (50021, 64, 1, False), (50021, 64, 4, True), (40009, 64, 16, False)])
def test_bdot_fast_matches_oracle(fast, port, n, k, p, glob):
    x, y = seeded(n, k, 201), seeded(n, k, 202)
    got = bk.bdot(x, y, cfg(k, p, glob), ctx=fast).data
    want = port.bdot(x, y, p, glob)
    bound = port.bdot(np.abs(x), np.abs(y), p, glob)  # sum |x||y| scale of the rounding error
    assert np.all(np.abs(got - want) <= 1e-13 * bound + 1e-300)


# --------------------------------------------------------------- BAXPY ---
def test_baxpy_zero_coefficient_leaves_x(ctx):
    x = seeded(5, 4, 1)
    before = x.copy()
    bk.baxpy(x, seeded(5, 4, 2), bk.BlockCoefficient(cfg(4, 2)), ctx=ctx)
    np.testing.assert_array_equal(x, before)


def test_baxpy_identity_adds(ctx):
    for glob in (False, True):
        x, y = seeded(5, 4, 1), seeded(5, 4, 2)
        before = x.copy()
        bk.baxpy(x, y, bk.BlockCoefficient.identity(cfg(4, 2, glob)), ctx=ctx)
        np.testing.assert_array_equal(x, before + y)


def test_baxpy_matches_dense_embedding(ctx, port):
    for glob in (False, True):
        c = cfg(4, 2, glob)
        x, y = seeded(5, 4, 31), seeded(5, 4, 32)
        gam = bk.BlockCoefficient(c, port.rng_symmetric(33, c.block_count() * 4))
        emb = np.zeros((4, 4))
        for g in range(2):
            emb[2 * g:2 * g + 2, 2 * g:2 * g + 2] = gam.block(0 if glob else g)
        want = x + y @ emb
        bk.baxpy(x, y, gam, ctx=ctx)
        np.testing.assert_allclose(x, want, atol=1e-14)


def test_baxpy_negated_restores(ctx, port):
    c = cfg(8, 4)
    x, y = seeded(16, 8, 41), seeded(16, 8, 42)
    before = x.copy()
    gam = bk.BlockCoefficient(c, port.rng_symmetric(43, 2 * 16))
    bk.baxpy(x, y, gam, ctx=ctx)
    bk.baxpy(x, y, gam.negated(), ctx=ctx)
    np.testing.assert_allclose(x, before, atol=1e-13)


@pytest.mark.parametrize("n,k,p,glob", [(7, 8, 2, True), (33, 6, 3, False), (5000, 16, 4, False),
                                        (5000, 64, 16, False), (5000, 64, 4, True),
                                        (5000, 32, 8, False)])
def test_baxpy_exact_is_bitwise_oracle(exact, port, n, k, p, glob):
    x, y = seeded(n, k, 51), seeded(n, k, 52)
    blocks = 1 if glob else k // p
    gam = port.rng_symmetric(53, blocks * p * p).reshape(blocks, p, p)
    want = port.baxpy(x, y, gam, p, glob)
    bk.baxpy(x, y, bk.BlockCoefficient(cfg(k, p, glob), gam), ctx=exact)
    assert x.tobytes() == want.tobytes()


def test_baxpy_flops(ctx):
    for n in (16, 25):
        for k in (4, 8):
            for p in (1, 2, 4, 8):
                if k % p:
                    continue
                for glob in (False, True):
                    f = bk.FlopCounter()
                    x, y = seeded(n, k, 81), seeded(n, k, 82)
                    bk.bdot(x, y, cfg(k, p, glob), f, ctx=ctx)
                    assert f.multiply_adds_bdot == 2 * n * p * p * (k // p)
                    bk.baxpy(y, x, bk.BlockCoefficient.identity(cfg(k, p, glob)), f, ctx=ctx)
                    assert f.multiply_adds_baxpy == 2 * n * p * p * (k // p)


# ----------------------------------------------------------------- BOP ---
def test_bop_identity_and_twice(ctx):
    x = seeded(6, 3, 51)
    eye = bk.SparseMatrix.from_triplets(6, [(i, i, 1.0) for i in range(6)])
    np.testing.assert_array_equal(bk.bop(eye, x, ctx=ctx), x)
    two = bk.SparseMatrix.from_triplets(6, [(i, i, 2.0) for i in range(6)])
    np.testing.assert_array_equal(bk.bop(two, x, ctx=ctx), 2.0 * x)


def test_bop_poisson_matches_dense(ctx):
    a = bk.poisson2d(bk.PoissonSpec.constant(4, 4))
    x = seeded(16, 4, 52)
    dense = np.zeros((16, 16))
    rp, cl, vl = a.row_offsets(), a.col_indices(), a.values()
    for r in range(16):
        for i in range(rp[r], rp[r + 1]):
            dense[r, cl[i]] = vl[i]
    np.testing.assert_allclose(bk.bop(a, x, ctx=ctx), dense @ x, atol=1e-13)
    f = bk.FlopCounter()
    a5 = bk.poisson2d(bk.PoissonSpec.constant(5, 5))
    bk.bop(a5, seeded(25, 4, 83), flops=f, ctx=ctx)
    assert f.multiply_adds_bop == 2 * 4 * a5.nnz()


@pytest.mark.parametrize("kind,dims,k", [(POISSON2D_LOGUNI, (5, 5, 1), 8),
                                         (POISSON2D_CONST, (64, 48, 1), 3),
                                         (3, (20, 20, 20), 32), (4, (17, 17, 17), 16),
                                         (3, (16, 16, 16), 64), (2, (128, 128, 1), 64)])
def test_bop_matches_oracle(ctx, port, kind, dims, k):
    a = bk.stencil(kind, *dims, seed=11)
    x = seeded(a.n(), k, 61)
    got = bk.bop(a, x, ctx=ctx)
    want = port.bop((a.row_offsets(), a.col_indices(), a.values()), x)
    if ctx.numerics == "exact":
        assert got.tobytes() == want.tobytes()
    else:
        scale = port.bop((a.row_offsets(), a.col_indices(), np.abs(a.values())), np.abs(x))
        assert np.all(np.abs(got - want) <= 1e-14 * scale)


# -------------------------------------------------------------- BSOLVE ---
def test_bsolve_identity_and_scalar(ctx, port):
    c = cfg(6, 3)
    delta = bk.BlockCoefficient(c, port.rng_symmetric(61, 18))
    out = bk.bsolve(bk.BlockCoefficient.identity(c), delta, ctx=ctx)
    np.testing.assert_array_equal(out.data, delta.data)
    c = cfg(4, 2)
    g = bk.BlockCoefficient(c)
    g.data[:] = 2.0 * np.eye(2)
    d = bk.BlockCoefficient(c, port.rng_symmetric(62, 8))
    np.testing.assert_array_equal(bk.bsolve(g, d, ctx=ctx).data, d.data / 2.0)


@pytest.mark.parametrize("k,p,glob", [(9, 3, False), (8, 8, False), (32, 8, False),
                                      (64, 16, False), (64, 1, False), (64, 4, True),
                                      (16, 16, False), (40, 20, False)])
def test_bsolve_bitwise_oracle_and_residual(ctx, port, k, p, glob):
    blocks = 1 if glob else k // p
    rng = np.random.default_rng(k * 100 + p)
    gam = np.empty((blocks, p, p))
    for b in range(blocks):
        g = rng.uniform(-1, 1, (p, p))
        gam[b] = g.T @ g + np.eye(p) + 0.1 * rng.uniform(-1, 1, (p, p))  # non-symmetric
    delta = rng.uniform(-1, 1, (blocks, p, p))
    c = cfg(k, p, glob)
    out = bk.bsolve(bk.BlockCoefficient(c, gam), bk.BlockCoefficient(c, delta), ctx=ctx)
    want, bad = port.bsolve(gam, delta, k, p, glob)
    assert bad is None
    assert out.data.tobytes() == want.tobytes()  # same LU op order in both modes
    for b in range(blocks):
        np.testing.assert_allclose(gam[b] @ out.data[b], delta[b], atol=1e-11)


def test_bsolve_singular_block_index(ctx):
    c = cfg(4, 2)
    g = bk.BlockCoefficient.identity(c)
    g.data[1] = [[1.0, 2.0], [1.0, 2.0]]
    with pytest.raises(bk.BreakdownError) as e:
        bk.bsolve(g, bk.BlockCoefficient.identity(c), ctx=ctx)
    assert e.value.block_index == 1
    g2 = bk.BlockCoefficient(cfg(8, 2))
    g2.data[:] = np.eye(2)
    g2.data[3] = 0.0
    g2.data[2] = [[1e-20, 0.0], [0.0, 1.0]]  # pivot below 1e-14 * max-norm
    with pytest.raises(bk.BreakdownError) as e:
        bk.bsolve(g2, bk.BlockCoefficient.identity(cfg(8, 2)), ctx=ctx)
    assert e.value.block_index == 2


# --------------------------------------------------------- column norms ---
def test_column_norms(ctx, port):
    np.testing.assert_array_equal(bk.column_norms(np.zeros((5, 3)), ctx=ctx), np.zeros(3))
    basis = np.zeros((6, 4))
    for c in range(4):
        basis[c, c] = 1.0
    np.testing.assert_array_equal(bk.column_norms(basis, ctx=ctx), np.ones(4))
    x = seeded(17, 5, 71)
    want = np.sqrt((x * x).sum(axis=0))
    np.testing.assert_allclose(bk.column_norms(x, ctx=ctx), want, rtol=1e-14)
    for n, k in ((17, 5), (100000, 8), (65536, 64), (4099, 16)):
        x = seeded(n, k, 72)
        got = bk.column_norms(x, ctx=ctx)
        ref = port.column_norms(x)
        if ctx.numerics == "exact":
            assert got.tobytes() == ref.tobytes()
        else:
            np.testing.assert_allclose(got, ref, rtol=1e-13)


def test_kernels_finite(ctx):
    c = cfg(4, 2)
    a = bk.poisson2d(bk.PoissonSpec.heterogeneous(4, 4, 5))
    x, y = seeded(16, 4, 91), seeded(16, 4, 92)
    g = bk.bdot(x, y, c, ctx=ctx)
    bk.baxpy(x, y, g, ctx=ctx)
    z = bk.bop(a, x, ctx=ctx)
    s = bk.bsolve(bk.bdot(x, x, c, ctx=ctx), g, ctx=ctx)
    assert np.all(np.isfinite(x)) and np.all(np.isfinite(z)) and np.all(np.isfinite(s.data))


def test_matrix_upload_validates_structure_on_device(ctx):
    # sparse_matrix.hpp:96-105 structural checks, enforced by bkg_matrix_create
    bad = [([0, 2, 1], [0, 1, 0], 3),        # offsets decrease
           ([0, 1, 2], [0, 5], 2),            # column out of range
           ([0, 2, 3], [1, 0, 1], 3)]         # columns not ascending
    for off, cols, nnz in bad:
        a = bk.SparseMatrix(len(off) - 1, np.array(off, np.uint64)[: len(off)],
                            np.array(cols, np.uint64), np.ones(len(cols)), validate=False)
        with pytest.raises(bk.ConfigError):
            bk.bop(a, np.ones((a.n(), 2)), ctx=ctx)
