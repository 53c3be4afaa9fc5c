"""Multi-GPU path, host logic, on CPU: two processes over the gloo backend
(world_size 2) each take a row slab of a 3D stencil, derive the operand rows
they need, exchange ranges (all_gather), build the halo plan through the C
ABI (bkg_halo_plan) and check it: every ghost row arrives exactly once, each
rank's sends equal its peers' receives, and a halo-exchanged partitioned SpMM
(numpy stand-in for the device kernels) equals the global product; the
per-rank Gram partials sum to the global Gram (what the NCCL allreduce
combines)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1912_11930_b200 as bk
from paper_1912_11930_b200.partitioned import halo_plan, local_csr, need_range, row_blocks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _dense_spmm(lrp, cols, vals, xext, lo, k):
    nloc = len(lrp) - 1
    y = np.zeros((nloc, k))
    for r in range(nloc):
        for i in range(int(lrp[r]), int(lrp[r + 1])):
            y[r] += vals[i] * xext[int(cols[i]) - lo]
    return y


def _worker(rank, world, port, kind, dims, k, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = bk.stencil(kind, *dims)
        n = a.n()
        rb = row_blocks(n, world)
        r0, r1 = rb[rank], rb[rank + 1]
        lrp, cols, vals = local_csr(a, r0, r1)
        lo, hi = need_range(r0, r1, cols)
        ranges = [None] * world
        dist.all_gather_object(ranges, (r0, r1, lo, hi))
        assert [r[0] for r in ranges] + [ranges[-1][1]] == rb
        plan = halo_plan(rb, [r[2] for r in ranges], [r[3] for r in ranges])
        plans = [None] * world
        dist.all_gather_object(plans, plan)
        assert all(p == plan for p in plans)  # identical on every rank
        # every needed foreign row is received exactly once
        got = np.zeros(hi - lo, dtype=int)
        for d, s, row, cnt in plan:
            if d == rank:
                assert s != rank and rb[s] <= row and row + cnt <= rb[s + 1]
                got[row - lo:row - lo + cnt] += 1
        got[r0 - lo:r1 - lo] += 1
        assert np.all(got == 1)
        # halo exchange of a global operand X, then the partitioned SpMM
        x = bk.normal_block_rhs(n, k, 3)
        xext = np.zeros((hi - lo, k))
        xext[r0 - lo:r1 - lo] = x[r0:r1]
        sends = {}
        for d, s, row, cnt in plan:
            if s == rank:
                sends[d] = sends.get(d, []) + [(row, x[row:row + cnt].copy())]
        box = [None] * world
        dist.all_gather_object(box, sends)
        for src, payload in enumerate(box):
            for row, blk in payload.get(rank, []):
                xext[row - lo:row - lo + blk.shape[0]] = blk
        y = _dense_spmm(lrp, cols, vals, xext, lo, k)
        rp, cg, vg = a.row_offsets(), a.col_indices(), a.values()
        yg = np.zeros((r1 - r0, k))
        for r in range(r0, r1):
            for i in range(int(rp[r]), int(rp[r + 1])):
                yg[r - r0] += vg[i] * x[int(cg[i])]
        np.testing.assert_allclose(y, yg, rtol=0, atol=1e-12)
        # Gram partials: their sum over ranks is the global Gram X^T A X
        parts = [None] * world
        dist.all_gather_object(parts, x[r0:r1].T @ y)
        ax = np.zeros((n, k))
        for r in range(n):
            for i in range(int(rp[r]), int(rp[r + 1])):
                ax[r] += vg[i] * x[int(cg[i])]
        err = float(np.abs(sum(parts) - x.T @ ax).max())
        assert err <= 1e-10 * float(np.abs(x.T @ ax).max())
        out_q.put((rank, err, len(plan)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,dims", [(3, (6, 5, 8)), (4, (5, 4, 7)), (2, (9, 12, 1))])
def test_gloo_two_rank_halo_plan(kind, dims):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, dims, 8, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert [r[0] for r in res] == [0, 1]
    assert all(r[2] == 2 for r in res)  # one copy each way between the two slabs


def test_halo_plan_three_parts_banded():
    # 1D tridiagonal-like bands: part r needs one row on each side
    rb = [0, 10, 20, 30]
    plan = halo_plan(rb, [0, 9, 19], [11, 21, 30])
    assert sorted(plan) == sorted([(0, 1, 10, 1), (1, 0, 9, 1), (1, 2, 20, 1), (2, 1, 19, 1)])
    # a part needing rows from a non-neighbour gets a copy from it too
    plan = halo_plan(rb, [0, 0, 5], [30, 30, 30])
    assert (2, 0, 5, 5) in plan and (0, 2, 20, 10) in plan
