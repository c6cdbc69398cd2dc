"""Full-size parity of the bench's exact launches (-m gpu) against the oracle's goldens.

tests/golden/fullsize.txt is written by tools/make_goldens.py, which calls only oracle/
on the seeded inputs bench.py times; here every launch plan bench.py measures must
reproduce it.  The EDM end-to-end call is checked on sampled rows
against the oracle computed on the spot, plus an every-cell-written check.
"""
import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import golden  # noqa: E402
from paper_1609_01490_b200 import inputs  # noqa: E402
from paper_1609_01490_b200 import tri  # noqa: E402

G = {k: v for k, v in golden("fullsize.txt")}


def T(r):
    return r * (r + 1) // 2


@pytest.fixture(scope="module", autouse=True)
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    tri.lib()


@pytest.fixture(scope="module")
def spheres():
    return torch.from_numpy(inputs.spheres(200000, 42, 0.01)).cuda()


# bench.py: SIMT filter at rho = 256 (lambda / persist / BB), tcgen05 at rho = 768 (lambda / BB)
@pytest.mark.parametrize("strategy,rho", [("lambda", 256), ("persist", 256), ("bb", 256), ("tc", 768),
                                          ("bb_tc", 768), ("tc", 256), ("tc", 512), ("tc", 1024)])
def test_collide_full_size_golden(spheres, strategy, rho):
    m = tri.tri_map_init(200000, rho, 1, 0, 1, 0)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_collide(m, strategy, spheres, cnt)
    torch.cuda.synchronize()
    assert cnt.item() == int(G["collide_n200000_seed42_r0.01"])


@pytest.mark.parametrize("strategy", ["lambda", "bb"])
def test_collide1d_full_size_golden(strategy):
    iv = torch.from_numpy(inputs.intervals(200000, 42, 1e-5)).cuda()
    m = tri.tri_map_init(200000, 256, 1, 0, 1, 1)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_collide1d(m, strategy, iv, cnt)
    torch.cuda.synchronize()
    assert cnt.item() == int(G["collide1d_n200000_seed42_r1e-5"])


def _digest(t):
    a = t.cpu().numpy()
    return hashlib.sha256(a.tobytes()).hexdigest(), int(a.sum(dtype=np.int64))


def _ca_plan(strategy, rho, plan):
    n = 32768
    m = tri.tri_map_init(n, rho)
    x = torch.from_numpy(inputs.ca_state(n, 42)).cuda()
    y = torch.empty_like(x)
    for k in plan:
        if k == 1 and rho == 128:
            tri.tri_ca_step(m, strategy, x, y)
        else:
            tri.tri_ca_steps(m, strategy, k, x, y)
        x, y = y, x
    torch.cuda.synchronize()
    return _digest(x)


@pytest.mark.parametrize("strategy", ["lambda", "bb"])
def test_ca_bench_plan_100_generations(strategy):
    """bench.py's plan: rho = 224 tiles, 12 launches of 8 generations + one of 4."""
    got = _ca_plan(strategy, 224, [8] * 12 + [4])
    assert got == (G["ca_n32768_seed42_g100_sha256"], int(G["ca_n32768_seed42_g100_alive"]))


@pytest.mark.parametrize("strategy", ["lambda", "persist", "bb"])
def test_ca_single_step_plan_100_generations(strategy):
    """bench.py's single-generation plan: tri_ca_step at rho = 128, 100 launches."""
    got = _ca_plan(strategy, 128, [1] * 100)
    assert got == (G["ca_n32768_seed42_g100_sha256"], int(G["ca_n32768_seed42_g100_alive"]))


@pytest.mark.parametrize("strategy", ["lambda", "bb"])
def test_ca_run_packed_100_generations(strategy):
    """tri_ca_run, the bench's CA path: the bit-packed state, 13 launches of <= 8 generations."""
    n = 32768
    m = tri.tri_map_init(n, 240)
    x = torch.from_numpy(inputs.ca_state(n, 42)).cuda()
    y = torch.empty_like(x)
    tri.tri_ca_run(m, strategy, 100, x, y)
    torch.cuda.synchronize()
    assert _digest(y) == (G["ca_n32768_seed42_g100_sha256"], int(G["ca_n32768_seed42_g100_alive"]))
    tri.tri_ca_run(m, "lambda", 8, x, y)
    torch.cuda.synchronize()
    assert _digest(y) == (G["ca_n32768_seed42_g8_sha256"], int(G["ca_n32768_seed42_g8_alive"]))


@pytest.mark.parametrize("rho,k", [(224, 8), (128, 8), (128, 1)])
def test_ca_first_launch(rho, k):
    got = _ca_plan("lambda", rho, [k])
    g = 8 if k == 8 else 1
    assert got == (G[f"ca_n32768_seed42_g{g}_sha256"], int(G[f"ca_n32768_seed42_g{g}_alive"]))


@pytest.mark.parametrize("strategy", ["lambda", "persist", "bb"])
def test_triplet_full_size_total(strategy):
    """bench.py's triplet launch (n = 4096, rho = 32): the total energy within the
    normalised tolerance of reading Q15, 1e-5 * sum |E|."""
    x = torch.from_numpy(inputs.points4(4096, 42)).cuda()
    tm = tri.tet_map_init(4096, 32)
    e = torch.empty(4096, dtype=torch.float64, device="cuda")
    tri.tet_triplet(tm, strategy, x, e)
    torch.cuda.synchronize()
    total, absum = float(G["triplet_n4096_seed42_total"]), float(G["triplet_n4096_seed42_abs"])
    assert abs(e.sum().item() - total) <= 1e-5 * absum


def test_edm_host_bench_config(orc):
    """tri_edm_host exactly as bench.py's e2e leg calls it: lambda, rho = 128, 2^25-cell
    bands, n = 65536, pinned host buffers.  Every cell is written (the host buffer starts
    as NaN) and sampled rows -- first, last, band edges, random -- match the oracle."""
    n = 65536
    pts_h = inputs.points(n, 3, 42)
    m = tri.tri_map_init(n, 128)
    h_pts = torch.from_numpy(pts_h).pin_memory()
    h_out = torch.empty(m.out_cells, dtype=torch.float32, pin_memory=True)
    h_out.fill_(float("nan"))
    band = 1 << 25
    ws = torch.empty(2 * 4 * band + 64, dtype=torch.uint8, device="cuda")
    d_pts = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    tri.tri_edm_host(m, "lambda", h_pts, d_pts, h_out, ws, band)
    out = h_out.numpy()
    assert not np.isnan(out).any()
    rng = np.random.default_rng(1)
    rows = sorted({0, 1, 127, 128, 511, 512, n - 129, n - 128, n - 1, *rng.integers(0, n, 12).tolist()})
    for r in rows:
        ref = orc.edm(pts_h, r, r + 1)
        got = out[T(r):T(r) + r + 1]
        assert np.all(np.abs(got - ref) <= np.maximum(1e-5 * np.abs(ref), 1e-6)), r


@pytest.mark.parametrize("strategy", ["lambda", "bb"])
def test_edm_tile_row_past_2_25(orc, strategy):
    """One tile row of an n = 2^25 + 1000 EDM (rows [r0, r0 + 128), r0 = 262145 * 128 > 2^25,
    each row ~33.5 M cells; 17.2 GB of output): the line-owned interior tiles' 64-bit row
    pointer path (taken only for r0 >= 2^25) and the diagonal tiles' checked path at 64-bit
    offsets.  The map is the snapped slice of that tile row (row and omega range set by hand);
    every cell is written and rows covering all four members of a same-phase quad, both walk
    ends and the diagonal tile match the oracle."""
    rho, bi = 128, 262145
    n = (1 << 25) + 1000
    r0 = bi * rho
    assert r0 >= (1 << 25) and r0 + rho <= n
    m = tri.tri_map_init(n, rho)
    m.world, m.rank, m.snap = 2, 1, 1
    m.row_begin, m.row_end = r0, r0 + rho
    m.omega_begin, m.omega_end = T(bi), T(bi + 1)
    m.out_offset, m.out_cells = T(r0), T(r0 + rho) - T(r0)
    pts_h = inputs.points(n, 3, 7)
    pts = torch.from_numpy(pts_h).cuda()
    out = torch.full((m.out_cells,), float("nan"), dtype=torch.float32, device="cuda")
    tri.tri_edm(m, strategy, pts, out)
    torch.cuda.synchronize()
    assert not torch.isnan(out).any().item()                       # every cell of the slice written
    for y in (0, 1, 31, 32, 63, 64, 95, 96, 126, 127):            # quads {x, 63-x, 64+x, 127-x}
        r = r0 + y
        got = out[T(r) - m.out_offset:T(r) - m.out_offset + r + 1].cpu().numpy()
        ref = orc.edm(pts_h, r, r + 1)
        assert np.all(np.abs(got - ref) <= np.maximum(1e-5 * np.abs(ref), 1e-6)), y
    del out
