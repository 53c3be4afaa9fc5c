"""Product input generators (libbkgpu.so host code) == oracle, bit for bit.

poisson2d / random_block_rhs restate problems.hpp:74-134 (pinned to the
reference in test_oracle.py); the N(0,1), lognormal and 3D stencil
generators are the frozen synthetic inputs of DESIGN.md §Inputs.
"""
import numpy as np
import pytest

import paper_1912_11930_b200 as bk
from cases import (DIFFUSION2D_LOGNORMAL, LAPLACE3D_7PT, POISSON2D_CONST, POISSON2D_LOGUNI,
                   STENCIL3D_27PT)


@pytest.mark.parametrize("kind,dims", [
    (POISSON2D_CONST, (2, 2, 1)), (POISSON2D_CONST, (7, 5, 1)), (POISSON2D_LOGUNI, (16, 16, 1)),
    (DIFFUSION2D_LOGNORMAL, (9, 13, 1)), (LAPLACE3D_7PT, (2, 2, 2)), (LAPLACE3D_7PT, (5, 4, 3)),
    (STENCIL3D_27PT, (2, 2, 2)), (STENCIL3D_27PT, (6, 5, 4))])
def test_stencil_matches_oracle(port, kind, dims):
    nx, ny, nz = dims
    a = bk.stencil(kind, nx, ny, nz, seed=11, contrast=2.0, validate=True)
    rp, cols, vals = port.stencil(kind, nx, ny, nz, seed=11, contrast=2.0)
    assert a.row_offsets().tobytes() == rp.tobytes()
    assert a.col_indices().tobytes() == cols.tobytes()
    assert a.values().tobytes() == vals.tobytes()


def test_stencil_shapes_match_baseline_configs():
    # nnz of the full-size configs, from the closed forms
    import ctypes as C
    from paper_1912_11930_b200 import _native as N
    for kind, dims, n_exp, z_exp in [
            (POISSON2D_CONST, (128, 128, 1), 16384, 81408),
            (LAPLACE3D_7PT, (128, 128, 128), 2097152, 14581760),
            (DIFFUSION2D_LOGNORMAL, (1024, 1024, 1), 1048576, 5238784),
            (STENCIL3D_27PT, (192, 192, 192), 7077888, 189119224),
            (LAPLACE3D_7PT, (384, 384, 384), 56623104, 395476992),
            (LAPLACE3D_7PT, (256, 256, 256), 16777216, 117047296)]:
        n, z = C.c_uint64(), C.c_uint64()
        assert N.lib().bkg_stencil_size(kind, *dims, C.byref(n), C.byref(z)) == 0
        assert (n.value, z.value) == (n_exp, z_exp)


def test_rhs_generators_match_oracle(port):
    assert bk.random_block_rhs(33, 7, 5).tobytes() == port.random_block_rhs(33, 7, 5).tobytes()
    assert bk.normal_block_rhs(33, 7, 5).tobytes() == port.normal_block_rhs(33, 7, 5).tobytes()
    z = bk.normal_block_rhs(4096, 64, 7)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01


def test_poisson2d_validates_like_reference():
    with pytest.raises(bk.ConfigError):
        bk.poisson2d(bk.PoissonSpec.constant(1, 4))
    a = bk.poisson2d(bk.PoissonSpec.constant(4, 4))
    assert a.n() == 16 and a.nnz() == 64
    assert a.at(5, 5) == 4.0 and a.at(5, 6) == -1.0 and a.at(0, 15) == 0.0


# The product generators run in parallel chunks of >= 2^18 draws started from
# jumped Xorshift64Star states (csrc/rng.h); the oracle is serial.
@pytest.mark.parametrize("n,k", [(262143, 1), (262145, 3), (300001, 5)])
def test_parallel_uniform_rhs_matches_serial_oracle(port, n, k):
    assert bk.random_block_rhs(n, k, 9).tobytes() == port.random_block_rhs(n, k, 9).tobytes()


@pytest.mark.parametrize("n,k", [(524289, 1), (200001, 5)])
def test_parallel_normal_rhs_matches_serial_oracle(port, n, k):
    assert bk.normal_block_rhs(n, k, 13).tobytes() == port.normal_block_rhs(n, k, 13).tobytes()


@pytest.mark.parametrize("kind", [POISSON2D_LOGUNI, DIFFUSION2D_LOGNORMAL])
def test_parallel_coefficient_fields_match_serial_oracle(port, kind):
    a = bk.stencil(kind, 777, 701, 1, seed=4, contrast=1.5)  # 544,677 cells
    rp, cols, vals = port.stencil(kind, 777, 701, 1, seed=4, contrast=1.5)
    assert a.values().tobytes() == vals.tobytes()


def test_jump_ahead_matches_stepping(port):
    # position m of the stream from a jumped state == the m-th serial draw
    full = port.random_block_rhs(1, 1_000_003, 21).ravel()
    chunk = bk.random_block_rhs(1, 1_000_003, 21).ravel()
    assert chunk.tobytes() == full.tobytes()
