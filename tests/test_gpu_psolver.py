"""Row-partitioned solver on one B200: `nparts` virtual parts (the single-GPU
emulation of nparts ranks: halo copies + fixed-order allreduce), and the NCCL
transport with one rank.  Checked against the reference fixtures / oracle
with the north_star bars, and against the unpartitioned solver."""
import numpy as np
import pytest

import golden_io
import paper_1912_11930_b200 as bk
from cases import BY_NAME, build_inputs
from paper_1912_11930_b200.partitioned import PartitionedSolver, local_csr, nccl_unique_id

pytestmark = pytest.mark.gpu


class Gen:
    def stencil(self, kind, nx, ny, nz=1, seed=0, contrast=2.0):
        a = bk.stencil(kind, nx, ny, nz, seed=seed, contrast=contrast)
        return a.row_offsets(), a.col_indices(), a.values()

    normal_block_rhs = staticmethod(bk.normal_block_rhs)
    random_block_rhs = staticmethod(bk.random_block_rhs)


@pytest.fixture(scope="module")
def ctx():
    c = bk.Context(0, "fast")
    yield c
    c.close()


def inputs(name):
    case = BY_NAME[name]
    csr, b, _ = build_inputs(case, Gen())
    a = bk.SparseMatrix(len(csr[0]) - 1, *csr, validate=False)
    return case, a, b


@pytest.mark.parametrize("name", ["c2_24", "c4_14_classical", "c4_14_hybrid4", "c4_14_global4",
                                  "c5_16", "c1_classical", "c1_parallel"])
@pytest.mark.parametrize("nparts", [1, 2, 3, 4])
def test_virtual_parts_meet_parity_bars(ctx, port, name, nparts):
    case, a, b = inputs(name)
    g = golden_io.load(name)
    cfg = bk.SubalgebraConfig(case.k, case.p, case.mode)
    s = PartitionedSolver.virtual(a, cfg, nparts, ctx)
    s.set_rhs(b)
    rep, fin = s.run(case.tol, case.max_iter, record_history=True, final_norms=True)
    hist = s.history(rep.history_rows)
    x = s.x()
    s.close()
    m = g["meta"]
    assert rep.converged == m["converged"]
    assert abs(rep.iterations - m["iterations"]) <= 1
    rows = min(len(hist), len(g["history"]))
    drift = np.max(np.abs(hist[:rows] - g["history"][:rows]) / g["history"][:rows])
    assert drift <= 1e-9, drift
    ref = port.bcg_solve((a.row_offsets(), a.col_indices(), a.values()), b, case.p, case.glob,
                         tol=case.tol, max_iter=case.max_iter, record_history=False)
    xs = np.linalg.norm(x - ref.x, axis=0) / np.linalg.norm(ref.x, axis=0)
    assert np.max(xs) <= 1e-8
    np.testing.assert_allclose(fin, ref.final_norms, rtol=1e-6, atol=1e-12)
    assert rep.flops_bdot == m["flops_bdot"] and rep.flops_bop == m["flops_bop"]


def test_nccl_single_rank_matches_virtual(ctx):
    case, a, b = inputs("c2_24")
    cfg = bk.SubalgebraConfig(case.k, case.p, case.mode)
    lrp, cols, vals = local_csr(a, 0, a.n())
    s = PartitionedSolver.nccl(a.n(), 0, a.n(), lrp, cols, vals, cfg, 0, 1, nccl_unique_id(), ctx)
    s.set_rhs(b)
    rep, _ = s.run(case.tol, case.max_iter, record_history=True)
    xn, hn = s.x(), s.history(rep.history_rows)
    s.close()
    v = PartitionedSolver.virtual(a, cfg, 1, ctx)
    v.set_rhs(b)
    rep1, _ = v.run(case.tol, case.max_iter, record_history=True)
    assert rep.iterations == rep1.iterations
    assert hn.tobytes() == v.history(rep1.history_rows).tobytes()  # same kernels, same order
    assert xn.tobytes() == v.x().tobytes()
    v.close()


def test_partitioned_breakdown_and_maxiter(ctx):
    case, a, b = inputs("c2_24")
    b = b.copy()
    b[:, 5] = b[:, 1]  # duplicate column inside p-group 0 -> singular alpha block 0
    s = PartitionedSolver.virtual(a, bk.SubalgebraConfig(32, 8), 3, ctx)
    s.set_rhs(b)
    rep, _ = s.run(1e-8, 0)
    assert rep.breakdown == 1 and rep.breakdown_iteration == 1 and rep.breakdown_block == 0
    s.close()
    s = PartitionedSolver.virtual(a, bk.SubalgebraConfig(32, 8), 2, ctx)
    s.set_rhs(bk.normal_block_rhs(a.n(), 32, 7))
    rep, _ = s.run(1e-30, 5)
    assert rep.iterations == 5 and not rep.converged
    s.close()


def test_generated_slab_rhs_matches_host_generator(ctx):
    """bkg_psolver_generate_rhs: every part generates its rows of B with the
    stream jumped to its first row -- U(-1,1) bit-identical to the host
    random_block_rhs over all n rows."""
    case, a, b = inputs("c2_24")
    s = PartitionedSolver.virtual(a, bk.SubalgebraConfig(32, 8), 3, ctx)
    s.generate_rhs("uniform", 7)
    assert s.rhs().tobytes() == bk.random_block_rhs(a.n(), 32, 7).tobytes()
    s.generate_rhs("normal", 7)
    np.testing.assert_allclose(s.rhs(), bk.normal_block_rhs(a.n(), 32, 7), rtol=1e-13, atol=1e-13)
    s.close()


@pytest.mark.parametrize("kind,grid,k,p", [(3, (24, 20, 18), 32, 8), (4, (14, 12, 13), 16, 4),
                                           (2, (40, 36, 1), 64, 1)])
def test_nccl_generated_matches_host_csr(ctx, kind, grid, k, p):
    """One rank, device-generated CSR (bkg_psolver_create_nccl_generated) vs
    the host CSR of the same stencil: same kernels, same bits."""
    nx, ny, nz = grid
    a = bk.stencil(kind, nx, ny, nz, seed=11 if kind == 2 else 0)
    n = a.n()
    cfg = bk.SubalgebraConfig(k, p)
    g = PartitionedSolver.nccl_generated(kind, nx, ny, nz, 0, n, cfg, 0, 1, nccl_unique_id(), ctx,
                                         rhs="uniform", seed=7,
                                         coeff_seed=11 if kind == 2 else 0)
    b = g.rhs()
    assert b.tobytes() == bk.random_block_rhs(n, k, 7).tobytes()
    rep, _ = g.run(1e-300, 12, record_history=True)
    xg, hg = g.x(), g.history(rep.history_rows)
    g.close()
    lrp, cols, vals = local_csr(a, 0, n)
    h = PartitionedSolver.nccl(n, 0, n, lrp, cols, vals, cfg, 0, 1, nccl_unique_id(), ctx)
    h.set_rhs(b)
    rep1, _ = h.run(1e-300, 12, record_history=True)
    assert rep.iterations == rep1.iterations == 12
    assert rep.flops_bop == rep1.flops_bop
    assert hg.tobytes() == h.history(rep1.history_rows).tobytes()
    assert xg.tobytes() == h.x().tobytes()
    h.close()


@pytest.mark.parametrize("nparts", [2, 3])
@pytest.mark.parametrize("stage", ["1", "0"])
def test_interior_boundary_split(ctx, monkeypatch, nparts, stage):
    """k1_stage in the partitioned loop: every part's blocks are split into
    interior blocks (launched while the halo copies run on the side stream)
    and boundary blocks (after the halo event); their alpha partials are
    summed in a fixed order.  Bars against the unpartitioned fast solve, and
    the split itself: a z-slab part of a 7-point stencil has boundary blocks
    only next to its neighbours (one plane each) and no ghost reads inside."""
    monkeypatch.setenv("BKG_K1_STAGE", stage)
    monkeypatch.setenv("BKG_K1_GRID", "0")
    case, a, b = inputs("c2_24")
    cfg = bk.SubalgebraConfig(case.k, case.p, case.mode)
    s = PartitionedSolver.virtual(a, cfg, nparts, ctx)
    plane = 24 * 24
    for i in range(nparts):
        info = s.part_info(i)
        if stage == "1":
            assert info["k1"] == "k1_stage"
            r0, r1 = info["rows"]
            nb = info["interior_blocks"] + info["boundary_blocks"]
            nbrs = (i > 0) + (i < nparts - 1)
            bx, by, bz = info["box"]
            if bx:  # grid boxes: only the box layers next to a neighbour read ghosts
                per_layer = -(-24 // bx) * -(-24 // by)
                layers = -(-((r1 - r0) // plane) // bz)
                assert nb == per_layer * layers
                assert 0 < info["boundary_blocks"] <= min(nbrs, layers) * per_layer
                assert info["interior_blocks"] == nb - info["boundary_blocks"]
                if layers > nbrs:
                    assert info["interior_blocks"] > 0
            else:   # consecutive rows: one plane of blocks per neighbour
                R = info["block_rows"]
                assert 0 < info["boundary_blocks"] <= nbrs * (-(-plane // R) + 1)
                assert info["interior_blocks"] > 0
        else:
            assert info["k1"] in ("k1_wide", "k1_line")
    s.set_rhs(b)
    rep, _ = s.run(1e-300, 40, record_history=True)
    hist, x = s.history(rep.history_rows), s.x()
    s.close()
    ref = bk.bcg_solve(a, b, bk.Preconditioner.identity(a.n()), cfg,
                       bk.SolveOptions(tol=1e-300, max_iter=40, record_history=True), ctx=ctx)
    h1 = np.array(ref.report.defect_history)
    assert rep.iterations == ref.report.iterations == 40
    assert np.max(np.abs(hist - h1) / h1) <= 1e-9
    xr = np.linalg.norm(x - ref.x, axis=0) / np.linalg.norm(ref.x, axis=0)
    assert np.max(xr) <= 1e-9


@pytest.mark.parametrize("kind,dims,k,p,mode", [(3, (24, 24, 24), 32, 8, "hybrid"),
                                                (4, (18, 16, 12), 16, 16, "hybrid"),
                                                (4, (18, 16, 12), 16, 4, "global"),
                                                (3, (20, 17, 8), 64, 16, "hybrid")])
@pytest.mark.parametrize("nparts", [1, 2, 4])
def test_grid_parts(ctx, monkeypatch, kind, dims, k, p, mode, nparts):
    """k1_grid in the partitioned loop (kernels_grid.cuh): a part that is whole
    z-planes of a constant-coefficient stencil reads its ghost-extended P as
    a (column, x, y, plane) tensor; planes that need no ghost plane are
    launched while the halo copies run, the one or two end planes after them.
    Bars against the unpartitioned fast solve with the CSR K1."""
    monkeypatch.setenv("BKG_K1_GRID", "1")
    monkeypatch.setenv("BKG_RESIDENT", "0")
    a = bk.stencil(kind, *dims, seed=11)
    n = a.n()
    b = bk.normal_block_rhs(n, k, 7)
    cfg = bk.SubalgebraConfig(k, p, mode)
    s = PartitionedSolver.virtual(a, cfg, nparts, ctx)
    plane = dims[0] * dims[1]
    tiles = -(-dims[0] // 16) * -(-dims[1] // 16) * (k // 16)
    for i in range(nparts):
        info = s.part_info(i)
        r0, r1 = info["rows"]
        if r0 % plane or r1 % plane:  # not whole planes: the CSR kernels
            assert info["k1"] != "k1_grid"
            continue
        assert info["k1"] == "k1_grid"
        nbrs = (i > 0) + (i < nparts - 1)
        planes = (r1 - r0) // plane
        assert info["boundary_blocks"] == tiles * min(nbrs, planes)  # one plane per neighbour
        assert (info["interior_blocks"] > 0) == (planes > nbrs)
    s.set_rhs(b)
    rep, _ = s.run(1e-300, 30, record_history=True)
    hist, x = s.history(rep.history_rows), s.x()
    s.close()
    monkeypatch.setenv("BKG_K1_GRID", "0")
    c2 = bk.Context(0, "fast")
    ref = bk.bcg_solve(a, b, bk.Preconditioner.identity(n), cfg,
                       bk.SolveOptions(tol=1e-300, max_iter=30, record_history=True), ctx=c2)
    c2.close()
    h1 = np.array(ref.report.defect_history)
    assert rep.iterations == ref.report.iterations == 30
    assert np.max(np.abs(hist - h1) / h1) <= 1e-9
    xr = np.linalg.norm(x - ref.x, axis=0) / np.linalg.norm(ref.x, axis=0)
    assert np.max(xr) <= 1e-9
