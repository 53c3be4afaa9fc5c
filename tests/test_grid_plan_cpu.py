"""Host logic of the grid-stencil K1's work plan (bkg_grid_plan; grid.cu
grid_plan / grid2_plan): pure arithmetic, no device.  Every plane (2-D: line)
of the requested range is produced by exactly one item per (tile, slice), the
persistent grid is a multiple of the k / 16 slices (a CTA keeps one slice)
and never exceeds the items, and the plan of a z-slab part is consistent with
its ghost-extended operand tensor."""
import ctypes as C

import pytest

from paper_1912_11930_b200 import _native as N

FIELDS = ("tiles_x", "tiles_y", "chunk", "nzc", "slices", "items", "ctas", "tmin", "tmax",
          "stride", "sync_every", "sync_lead")


def plan(nx, ny, nz, k, sms=148, zbeg=0, zend=None, zoff=0, nzt=None):
    zend = nz if zend is None else zend
    nzt = nz if nzt is None else nzt
    out = (C.c_int64 * 12)()
    rc = N.lib().bkg_grid_plan(nx, ny, nz, k, sms, zbeg, zend, zoff, nzt, out)
    assert rc == 0, N.lib().bkg_last_error()
    return dict(zip(FIELDS, [int(v) for v in out]))


@pytest.mark.parametrize("nx,ny,nz,k", [(256, 256, 256, 64), (128, 128, 128, 32),
                                        (192, 192, 192, 16), (33, 17, 9, 16), (6, 5, 4, 128),
                                        (384, 384, 48, 64), (16, 16, 1000, 16)])
def test_plan_covers_every_plane_once(nx, ny, nz, k):
    p = plan(nx, ny, nz, k)
    assert p["tiles_x"] == -(-nx // 16) and p["tiles_y"] == -(-ny // 16)
    assert p["slices"] == k // 16
    assert p["stride"] == p["chunk"] and p["nzc"] == -(-nz // p["chunk"])
    # items of one (tile, slice): [c * chunk, min((c + 1) * chunk, nz)) partition [0, nz)
    covered = []
    for c in range(p["nzc"]):
        covered += list(range(c * p["stride"], min(c * p["stride"] + p["chunk"], nz)))
    assert covered == list(range(nz))
    assert p["items"] == p["tiles_x"] * p["tiles_y"] * p["slices"] * p["nzc"]
    assert 0 < p["ctas"] <= min(148, p["items"]) and p["ctas"] % p["slices"] == 0
    assert (p["tmin"], p["tmax"]) == (0, nz - 1)


def test_plan_uses_the_machine():
    """The BASELINE shapes fill the 148 SMs: C5 within 2% of whole rounds, C4 in
    one round, and only long launches are paced."""
    c5 = plan(256, 256, 256, 64)
    rounds = -(-c5["items"] // c5["ctas"])
    assert c5["ctas"] == 148 and c5["items"] / (rounds * c5["ctas"]) > 0.98
    assert c5["sync_every"] > 0  # 28 rounds of 66 steps
    c4 = plan(192, 192, 192, 16)
    assert c4["items"] == c4["ctas"] == 144 and c4["sync_every"] == 0
    c2 = plan(128, 128, 128, 32)
    assert c2["ctas"] == 148 and c2["sync_every"] == 0


@pytest.mark.parametrize("nx,ny,k", [(1024, 1024, 64), (300, 257, 16), (128, 7, 32)])
def test_plan_2d_lines(nx, ny, k):
    p = plan(nx, ny, 1, k)
    assert p["tiles_x"] == -(-nx // 128) and p["tiles_y"] == 1
    covered = []
    for c in range(p["nzc"]):
        covered += list(range(c * p["stride"], min(c * p["stride"] + p["chunk"], ny)))
    assert covered == list(range(ny))
    assert p["items"] == p["tiles_x"] * p["slices"] * p["nzc"]
    assert 0 < p["ctas"] <= min(2 * 148, p["items"]) and p["ctas"] % p["slices"] == 0
    assert (p["tmin"], p["tmax"]) == (0, ny - 1)


def test_plan_of_a_z_slab_part():
    """A middle z-slab of 48 planes with both ghost planes: the interior launch
    produces planes [1, 47) and may read tensor planes 0 .. 49 (part coordinates
    -1 .. 48)."""
    p = plan(384, 384, 48, 64, zbeg=1, zend=47, zoff=1, nzt=50)
    assert (p["tmin"], p["tmax"]) == (-1, 48)
    covered = []
    for c in range(p["nzc"]):
        covered += list(range(1 + c * p["stride"], min(1 + c * p["stride"] + p["chunk"], 47)))
    assert covered == list(range(1, 47))


def test_plan_rejects_bad_shapes():
    out = (C.c_int64 * 12)()
    assert N.lib().bkg_grid_plan(16, 16, 16, 24, 148, 0, 16, 0, 16, out) != 0  # k % 16
    assert N.lib().bkg_grid_plan(16, 16, 16, 16, 148, 4, 4, 0, 16, out) != 0   # empty range
