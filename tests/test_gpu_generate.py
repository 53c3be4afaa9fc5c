"""Device-side problem generation (csrc/generate.cu)
against the host generators: stencils and the uniform RHS bit for bit, the
N(0,1) RHS within a few ulp (CUDA libm Box-Muller)."""
import numpy as np
import pytest

import paper_1912_11930_b200 as bk
from cases import (DIFFUSION2D_LOGNORMAL, LAPLACE3D_7PT, POISSON2D_CONST, POISSON2D_LOGUNI,
                   STENCIL3D_27PT)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = bk.Context(0, "exact")
    yield c
    c.close()


@pytest.mark.parametrize("kind,dims", [
    (POISSON2D_CONST, (2, 2, 1)), (POISSON2D_CONST, (7, 5, 1)), (POISSON2D_CONST, (128, 128, 1)),
    (POISSON2D_LOGUNI, (16, 16, 1)), (POISSON2D_LOGUNI, (300, 211, 1)),
    (DIFFUSION2D_LOGNORMAL, (9, 13, 1)), (DIFFUSION2D_LOGNORMAL, (1024, 257, 1)),
    (LAPLACE3D_7PT, (2, 2, 2)), (LAPLACE3D_7PT, (5, 4, 3)), (LAPLACE3D_7PT, (64, 33, 17)),
    (STENCIL3D_27PT, (2, 2, 2)), (STENCIL3D_27PT, (6, 5, 4)), (STENCIL3D_27PT, (31, 17, 9))])
def test_device_stencil_bitwise_host(ctx, kind, dims):
    nx, ny, nz = dims
    host = bk.stencil(kind, nx, ny, nz, seed=11, contrast=1.7)
    dev = bk.DeviceMatrix.generate(kind, nx, ny, nz, seed=11, contrast=1.7, ctx=ctx)
    assert (dev.n(), dev.nnz()) == (host.n(), host.nnz())
    d = dev.download()
    assert d.row_offsets().tobytes() == host.row_offsets().tobytes()
    assert d.col_indices().tobytes() == host.col_indices().tobytes()
    assert d.values().tobytes() == host.values().tobytes()
    dev.close()


@pytest.mark.parametrize("kind,dims", [(LAPLACE3D_7PT, (2, 2, 1)), (POISSON2D_CONST, (1, 5, 1)),
                                       (7, (4, 4, 4))])
def test_device_stencil_rejects_bad_shapes(ctx, kind, dims):
    with pytest.raises(bk.ConfigError):
        bk.DeviceMatrix.generate(kind, *dims, ctx=ctx)


@pytest.mark.parametrize("n,k", [(1, 1), (37, 3), (262145, 4), (1000003, 2)])
def test_device_uniform_rhs_bitwise_host(ctx, n, k):
    s = bk.DeviceSolver(_diag(n), bk.SubalgebraConfig(k, 1), ctx)
    s.generate_rhs("uniform", 17)
    assert s.rhs().tobytes() == bk.random_block_rhs(n, k, 17).tobytes()
    s.close()


def _diag(n):
    rp = np.arange(n + 1, dtype=np.uint64)
    return bk.SparseMatrix(n, rp, np.arange(n, dtype=np.uint64), np.ones(n), validate=False)


@pytest.mark.parametrize("n,k", [(5, 3), (262147, 2)])
def test_device_normal_rhs_within_ulps(ctx, n, k):
    s = bk.DeviceSolver(_diag(n), bk.SubalgebraConfig(k, 1), ctx)
    s.generate_rhs("normal", 7)
    got, want = s.rhs(), bk.normal_block_rhs(n, k, 7)
    np.testing.assert_allclose(got, want, rtol=4e-15, atol=4e-16)
    s.close()


def test_solve_on_device_generated_inputs_matches_host_inputs():
    # exact numerics: device matrix + device U(-1,1) RHS == host-generated inputs
    ctx = bk.Context(0, "exact")
    dev = bk.DeviceMatrix.generate(LAPLACE3D_7PT, 12, 11, 10, ctx=ctx)
    host = bk.stencil(LAPLACE3D_7PT, 12, 11, 10)
    cfg = bk.SubalgebraConfig(8, 4)
    s1 = bk.DeviceSolver(dev, cfg, ctx)
    s1.generate_rhs("uniform", 3)
    r1 = s1.run(1e-10, 0)
    s2 = bk.DeviceSolver(host, cfg, ctx)
    s2.set_rhs(bk.random_block_rhs(host.n(), 8, 3))
    r2 = s2.run(1e-10, 0)
    assert r1.iterations == r2.iterations and r1.converged
    assert s1.x().tobytes() == s2.x().tobytes()
    # the drop-in call accepts the device matrix too
    res = bk.bcg_solve(dev, bk.random_block_rhs(host.n(), 8, 3), bk.Preconditioner.identity(host.n()),
                       cfg, bk.SolveOptions(tol=1e-10), ctx=ctx)
    assert res.x.tobytes() == s2.x().tobytes()
    for s in (s1, s2):
        s.close()
    dev.close()
    ctx.close()


def test_device_matrix_bound_to_its_context():
    c1, c2 = bk.Context(0, "fast"), bk.Context(0, "fast")
    dev = bk.DeviceMatrix.generate(POISSON2D_CONST, 8, 8, ctx=c1)
    with pytest.raises(bk.ConfigError):
        bk.DeviceSolver(dev, bk.SubalgebraConfig(4, 4), c2)
    dev.close()
    c1.close()
    c2.close()
