"""GPU parity tests (-m gpu): the CUDA path through the C ABI against the CPU
oracle, element by element on the same seeded inputs.

Bars: bit-exact for indices, maps, dummy codes/digests/
counts, collision counts and CA states; EDM within 1e-5 relative (1e-6 absolute
near zero); triplet energies within 1e-5 of the per-particle scale
A_t = (1/3) sum |E| (reading Q15), total within 1e-5 of sum |E|.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1609_01490_b200 import inputs  # noqa: E402
from paper_1609_01490_b200 import tri  # noqa: E402

STRATS = ["lambda", "bb", "persist"]


def T(r):
    return r * (r + 1) // 2


@pytest.fixture(scope="module", autouse=True)
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    tri.lib()
    return torch.device("cuda:0")


def sync():
    torch.cuda.synchronize()


# ============================================================== map
def test_map_matches_enumeration(orc):
    m = 2000
    I, J = orc.enumerate_tri(m)
    cnt = len(I)
    ij = torch.empty(2 * cnt, dtype=torch.int32, device="cuda")
    fail = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_map_eval(0, cnt, ij, fail)
    sync()
    got = ij.cpu().numpy().astype(np.uint32).reshape(-1, 2)
    assert np.array_equal(got[:, 0], I) and np.array_equal(got[:, 1], J)
    assert fail.item() == 0


def test_map_exact_to_2_40_exhaustive():
    """Eq. 3 + successor rule for EVERY omega < 2^40 (the exactness bound)."""
    fail = torch.zeros(1, dtype=torch.int64, device="cuda")
    total = 0
    step = 1 << 38
    for w0 in range(0, 1 << 40, step):
        cnt = min(step, (1 << 40) - 1 - w0)   # successor of the last omega must stay < 2^40
        tri.tri_map_eval(w0, cnt, None, fail)
        sync()
        total += fail.item()
    assert total == 0


def test_map_boundaries_sampled(orc):
    ws = []
    for r in [1, 2, 3, 4607, 4608, 4609, 65535, 65536, 2**20, 1482908]:
        ws += [T(r) - 1, T(r), T(r) + 1]
    fail = torch.zeros(1, dtype=torch.int64, device="cuda")
    ij = torch.empty(2, dtype=torch.int32, device="cuda")
    for w in ws:
        tri.tri_map_eval(w, 1, ij, fail)
        sync()
        assert tuple(ij.cpu().numpy().astype(np.uint32).tolist()) == orc.lam(w)


def test_tet_map_matches_enumeration_and_exhaustive(orc):
    I, J, K = orc.enumerate_tet(120)
    cnt = len(I)
    ijk = torch.empty(3 * cnt, dtype=torch.int32, device="cuda")
    fail = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tet_map_eval(0, cnt, ijk, fail)
    sync()
    got = ijk.cpu().numpy().astype(np.uint32).reshape(-1, 3)
    assert np.array_equal(got[:, 0], I) and np.array_equal(got[:, 1], J) and np.array_equal(got[:, 2], K)
    assert fail.item() == 0
    total = 0
    step = 1 << 34
    for w0 in range(0, 1 << 36, step):
        tri.tet_map_eval(w0, step, None, fail)
        sync()
        total += fail.item()
    assert total == 0


# ============================================================== sqrt variants (section 4.1)
@pytest.mark.parametrize("variant,count", [(1, 12_000_000), (2, 2_000_000)])
def test_sqrt_variant_scan_matches_oracle(orc, variant, count):
    """lambda_X / lambda_N are IEEE-deterministic: the GPU's uncorrected variant
    fails at exactly the omegas the C oracle's fp32 restatement fails at."""
    fail = torch.zeros(1, dtype=torch.int64, device="cuda")
    first = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_map_eval_variant(variant, 0, count, fail, first)
    sync()
    nf, fw = orc.variant_scan(variant, 0, count)
    assert fail.item() == nf and first.item() == fw
    from conftest import golden
    g = {int(v): int(w) for v, _n, w in golden("sqrt_variants.txt")}
    assert first.item() == g[variant]           # SURVEY.md:38-40


def test_lambda_r_rows_within_rsqrtf_bound(orc):
    """lambda_R depends on the hardware rsqrtf, specified to 2 ulp (reading Q5c):
    every GPU row for omega < 2^23 lies in the oracle's reachable-row interval, and the GPU
    scan over [0, 2^24) fails on at least every surely-wrong and at most every maybe-wrong
    omega, no earlier than the first maybe-wrong one."""
    cnt = 1 << 23
    rows = torch.empty(cnt, dtype=torch.int32, device="cuda")
    tri.tri_map_rows_variant(tri.TRI_SQRT_R, 0, cnt, rows)
    sync()
    got = rows.cpu().numpy().astype(np.int64)
    lo, hi = orc.variant_r_rows(0, cnt)
    assert np.all(lo.astype(np.int64) <= got) and np.all(got <= hi.astype(np.int64))
    fail = torch.zeros(1, dtype=torch.int64, device="cuda")
    first = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_map_eval_variant(tri.TRI_SQRT_R, 0, 1 << 24, fail, first)
    sync()
    ns, fs, nm, fm = orc.variant_r_scan(0, 1 << 24)
    assert ns <= fail.item() <= nm
    if fail.item():
        assert first.item() >= fm and (fs is None or first.item() <= fs)


@pytest.mark.parametrize("variant", [1, 2])
def test_variant_rows_match_scan(orc, variant):
    """tri_map_rows_variant's lambda_X / lambda_N rows are the IEEE-deterministic ones: judged
    by Eq. 3 they fail exactly where the oracle scan says (count and first omega)."""
    cnt = 1 << 21
    rows = torch.empty(cnt, dtype=torch.int32, device="cuda")
    tri.tri_map_rows_variant(variant, 0, cnt, rows)
    sync()
    i = rows.cpu().numpy().astype(np.int64)
    w = np.arange(cnt, dtype=np.int64)
    bad = ~((i * (i + 1) // 2 <= w) & (w < (i + 1) * (i + 2) // 2))
    nf, fw = orc.variant_scan(variant, 0, cnt)
    assert int(bad.sum()) == nf and (int(w[np.argmax(bad)]) if bad.any() else None) == fw


def test_sqrt_variant_r_runs_and_dummy_variants():
    """The lambda_R scan runs; inside the first-failure bound the variant dummy kernels
    give the exact digest."""
    fail = torch.zeros(1, dtype=torch.int64, device="cuda")
    first = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_map_eval_variant(tri.TRI_SQRT_R, 0, 1 << 24, fail, first)
    sync()
    first_r = first.item() if fail.item() else 1 << 62
    n, rho = 2048, 16
    m = tri.tri_map_init(n, rho)
    assert m.blocks < 100_000 and m.blocks < first_r
    for s in ("lambda_x", "lambda_n", "lambda_r"):
        dig = torch.zeros(1, dtype=torch.int64, device="cuda")
        tri.tri_dummy(m, s, tri.TRI_DUMMY_DIGEST, dig)
        sync()
        assert dig.item() == (n - 1) * n * (n + 1) // 2


# ============================================================== dummy
@pytest.mark.parametrize("strategy", STRATS + ["rb"])
@pytest.mark.parametrize("n,rho", [(1, 8), (2, 16), (5, 8), (100, 16), (2048, 16), (1000, 32), (333, 8)])
def test_dummy_packed_digest_count(orc, strategy, n, rho):
    m = tri.tri_map_init(n, rho)
    out = torch.full((m.out_cells,), -1, dtype=torch.int32, device="cuda")
    tri.tri_dummy(m, strategy, tri.TRI_DUMMY_PACKED, out)
    sync()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), orc.dummy_packed(n))
    dig = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_dummy(m, strategy, tri.TRI_DUMMY_DIGEST, dig)
    sync()
    assert dig.item() == orc.dummy_digest(n) == (n - 1) * n * (n + 1) // 2
    cnt = torch.zeros(5, dtype=torch.int64, device="cuda")
    tri.tri_dummy(m, strategy, tri.TRI_DUMMY_COUNT, cnt)
    sync()
    c = cnt.cpu().tolist()
    ref = orc.dispatch_count(n, rho, {"bb": 1, "rb": 2}.get(strategy, 0))
    assert c == [ref["blocks"], ref["blocks_discarded"], ref["threads"], ref["useful"], ref["discarded"]]
    fx = torch.zeros(1, dtype=torch.int32, device="cuda")
    tri.tri_dummy(m, strategy, tri.TRI_DUMMY_FIXED, fx)
    sync()
    assert 0 <= fx.item() <= 2 * (n - 1)      # some in-domain i+j (racy by design, Q6)


def test_dummy_wide_codes(orc):
    n = 65600
    m = tri.tri_map_init(n, 32, 1, 7, 8, 1)   # last rank's slice: u64 codes
    out = torch.empty((m.out_cells,), dtype=torch.int64, device="cuda")
    tri.tri_dummy(m, "lambda", tri.TRI_DUMMY_PACKED, out)
    sync()
    ref = orc.dummy_packed(n, m.row_begin, m.row_end, elem_bytes=8)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), ref)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_dummy_ranks_concatenate(orc, world):
    n, rho = 777, 16
    parts = []
    for g in range(world):
        m = tri.tri_map_init(n, rho, 1, g, world, 1)
        out = torch.full((max(m.out_cells, 1),), -1, dtype=torch.int32, device="cuda")
        tri.tri_dummy(m, "lambda", tri.TRI_DUMMY_PACKED, out)
        sync()
        parts.append(out.cpu().numpy()[: m.out_cells].view(np.uint32))
    assert np.array_equal(np.concatenate(parts), orc.dummy_packed(n))


# ============================================================== EDM
def edm_close(got, ref):
    err = np.abs(got.astype(np.float64) - ref.astype(np.float64))
    tol = np.maximum(1e-5 * np.abs(ref.astype(np.float64)), 1e-6)
    bad = err > tol
    assert not bad.any(), (int(bad.sum()), float(err.max()))


@pytest.mark.parametrize("strategy", STRATS + ["rb", "clc"])
@pytest.mark.parametrize("rho", [32, 64, 128, 256])
@pytest.mark.parametrize("n,seed", [(1, 7), (2, 42), (3, 7), (5, 42), (64, 7), (257, 42), (1000, 7), (4097, 42)])
def test_edm_small(orc, strategy, rho, n, seed):
    pts = inputs.points(n, 3, seed)
    m = tri.tri_map_init(n, rho)
    out = torch.full((m.out_cells + 8,), float("nan"), dtype=torch.float32, device="cuda")
    tri.tri_edm(m, strategy, torch.from_numpy(pts).cuda(), out)
    sync()
    got = out.cpu().numpy()
    assert np.isnan(got[m.out_cells:]).all()        # nothing written past the slice
    edm_close(got[: m.out_cells], orc.edm(pts))


@pytest.mark.parametrize("rho", [128, 256])
@pytest.mark.parametrize("dim", [1, 2, 4])
def test_edm_dims_and_stride(orc, dim, rho):
    n = 777 if rho == 128 else 1601
    pts = inputs.points(n, dim, 7)
    m = tri.tri_map_init(n, rho)
    out = torch.empty((m.out_cells,), dtype=torch.float32, device="cuda")
    wide = torch.zeros((n, 6), dtype=torch.float32)
    wide[:, :dim] = torch.from_numpy(pts)
    tri.tri_edm(m, "lambda", wide.cuda()[:, :dim], out)      # ld = 6 > dim
    sync()
    edm_close(out.cpu().numpy(), orc.edm(pts))


@pytest.mark.parametrize("world,rho", [(2, 64), (3, 64), (5, 64), (3, 256), (4, 128)])
def test_edm_ranks_concatenate(orc, world, rho):
    n = 3001
    pts = inputs.points(n, 3, 42)
    d = torch.from_numpy(pts).cuda()
    parts = []
    for g in range(world):
        m = tri.tri_map_init(n, rho, 1, g, world, 1)
        out = torch.empty((max(m.out_cells, 4),), dtype=torch.float32, device="cuda")
        tri.tri_edm(m, "persist", d, out)
        sync()
        parts.append(out.cpu().numpy()[: m.out_cells])
    edm_close(np.concatenate(parts), orc.edm(pts))


@pytest.mark.parametrize("strategy,rho", [("lambda", 128), ("lambda", 256), ("persist", 128), ("clc", 128)])
def test_edm_full_size_sampled(orc, strategy, rho):
    """BASELINE configs[1]: n = 65536, 3-D; ("lambda", 128) is the bench's launch."""
    n = 65536
    pts = inputs.points(n, 3, 42)
    m = tri.tri_map_init(n, rho)
    out = torch.full((m.out_cells,), float("nan"), dtype=torch.float32, device="cuda")
    tri.tri_edm(m, strategy, torch.from_numpy(pts).cuda(), out)
    sync()
    assert not torch.isnan(out).any().item()           # every cell written
    for rb, re in [(0, 64), (20000, 20030), (40961, 40970), (65500, 65536)]:
        got = out[T(rb):T(re)].cpu().numpy()
        edm_close(got, orc.edm(pts, rb, re))
    del out


def test_edm_host_e2e(orc):
    n = 5000
    pts = torch.from_numpy(inputs.points(n, 3, 7))
    m = tri.tri_map_init(n, 128)
    h_out = torch.empty((m.out_cells,), dtype=torch.float32).pin_memory()
    ws = torch.empty((2 * 4 * 1_000_000,), dtype=torch.uint8, device="cuda")
    dp = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    tri.tri_edm_host(m, "persist", pts.pin_memory(), dp, h_out, ws, band_cells=1_000_000)
    edm_close(h_out.numpy(), orc.edm(pts.numpy()))


# ============================================================== collision
@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("rho", [128, 256, 512])
@pytest.mark.parametrize("n,seed,rmax", [(1, 7, 0.1), (2, 42, 0.9), (100, 7, 0.2), (1000, 42, 0.05),
                                         (5000, 7, 0.02), (777, 42, 0.08)])
def test_collide_small(orc, strategy, rho, n, seed, rmax):
    s = inputs.spheres(n, seed, rmax)
    m = tri.tri_map_init(n, rho)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_collide(m, strategy, torch.from_numpy(s).cuda(), cnt)
    sync()
    assert cnt.item() == orc.collide(s)


def test_collide_quantized_and_ranks(orc):
    s = inputs.spheres_quantized(20000, 42, 11, 0.01)
    d = torch.from_numpy(s).cuda()
    ref = orc.collide(s)
    tot = 0
    for g in range(3):
        m = tri.tri_map_init(20000, 128, 1, g, 3, 0)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        tri.tri_collide(m, "lambda", d, cnt)
        sync()
        tot += cnt.item()
    assert tot == ref


def _near_touching(n, seed, offset, scale):
    """n/2 random spheres and, n/2 indices later, a partner at distance (r_i + r_j)(1 + delta),
    delta within a few fp32 ulps of 0 (both signs): pairs on the predicate's knife edge, in
    off-diagonal tiles, around an offset origin (large |x| stresses the filter's margin)."""
    rng = np.random.default_rng(seed)
    h = n // 2
    c = rng.random((h, 3)) * scale + offset
    r = rng.random(h) * 0.01 * scale
    rp = rng.random(h) * 0.01 * scale
    d = rng.normal(size=(h, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    delta = rng.integers(-8, 9, size=h) * 2.0 ** -24
    p = c + d * ((r + rp) * (1 + delta))[:, None]
    s = np.zeros((2 * h, 4), np.float32)
    s[:h, :3], s[:h, 3] = c, r
    s[h:, :3], s[h:, 3] = p, rp
    return s


@pytest.mark.parametrize("offset,scale", [(0.0, 1.0), (0.5, 1.0), (100.0, 1.0), (-1000.0, 10.0), (0.0, 1e-3)])
def test_collide_knife_edge_pairs(orc, offset, scale):
    """The hot loop only filters (a 4-D dot-product gap with a rounding margin) and
    recounts flagged blocks with the fixed-order predicate: pairs within a few ulps of
    touching, at any coordinate magnitude, must be counted exactly as the oracle does."""
    s = _near_touching(8192, 11, offset, scale)
    ref = orc.collide(s)
    assert ref > 100            # the construction really puts pairs on both sides of the edge
    d = torch.from_numpy(s).cuda()
    for rho in (128, 256, 512):
        for strategy in STRATS:
            m = tri.tri_map_init(len(s), rho)
            cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
            tri.tri_collide(m, strategy, d, cnt)
            sync()
            assert cnt.item() == ref, (rho, strategy)


@pytest.mark.parametrize("strategy", ["tc", "bb_tc"])
@pytest.mark.parametrize("rho", [256, 384, 512, 640, 1024])
@pytest.mark.parametrize("n,seed,rmax", [(1, 7, 0.1), (300, 42, 0.2), (1000, 42, 0.05), (5000, 7, 0.02),
                                         (777, 42, 0.08), (1153, 7, 0.3)])
def test_collide_tc_small(orc, n, seed, rmax, rho, strategy):
    """TRI_LAMBDA_TC / TRI_BB_TC: the filter on the tensor cores (one tcgen05 tf32 MMA per
    128 x 128 block, TF32-exact operands), exact count."""
    s = inputs.spheres(n, seed, rmax)
    m = tri.tri_map_init(n, rho)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_collide(m, strategy, torch.from_numpy(s).cuda(), cnt)
    sync()
    assert cnt.item() == orc.collide(s)


@pytest.mark.parametrize("strategy", ["tc", "bb_tc"])
@pytest.mark.parametrize("rho", [256, 384, 512, 768, 1024])
@pytest.mark.parametrize("offset,scale", [(0.0, 1.0), (0.5, 1.0), (100.0, 1.0), (-1000.0, 10.0), (0.0, 1e-3),
                                          (0.49, 1e-4), (3.0, 0.1)])
def test_collide_tc_knife_edge(orc, offset, scale, rho, strategy):
    s = _near_touching(8192, 11, offset, scale)
    m = tri.tri_map_init(len(s), rho)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_collide(m, strategy, torch.from_numpy(s).cuda(), cnt)
    sync()
    assert cnt.item() == orc.collide(s)


def test_collide_tc_full_size_rank_slice(orc):
    n = 200000
    s = inputs.spheres(n, 42)
    d = torch.from_numpy(s).cuda()
    for g, rho in ((0, 256), (40, 256), (0, 512), (20, 512), (30, 384), (0, 1024), (9, 1024)):
        m = tri.tri_map_init(n, rho, 1, g, {256: 256, 384: 170, 512: 128, 1024: 64}[rho], 1)   # snapped rows
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        tri.tri_collide(m, "tc", d, cnt)
        sync()
        assert cnt.item() == orc.collide(s, m.row_begin, m.row_end)


@pytest.mark.parametrize("rho", [256, 384, 512, 1024])
def test_collide_tc_plain_ranks(orc, rho):
    """tcgen05 filter on plain (unsnapped) omega ranges of 3 ranks: the partial counts sum
    to the oracle's total (11-bit-quantised spheres: every fp32 op exact)."""
    n = 20000
    s = inputs.spheres_quantized(n, 42, 11, 0.01)
    d = torch.from_numpy(s).cuda()
    tot = 0
    for g in range(3):
        m = tri.tri_map_init(n, rho, 1, g, 3, 0)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        tri.tri_collide(m, "tc", d, cnt)
        sync()
        tot += cnt.item()
    assert tot == orc.collide(s)


def test_collide_full_size_rank_slice(orc):
    """BASELINE configs[2] (n = 200000): one 64-way snapped rank slice vs the oracle rows."""
    n = 200000
    s = inputs.spheres(n, 42)
    d = torch.from_numpy(s).cuda()
    for g in (0, 40):
        m = tri.tri_map_init(n, 256, 1, g, 256, 1)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        tri.tri_collide(m, "persist", d, cnt)
        sync()
        assert cnt.item() == orc.collide(s, m.row_begin, m.row_end)


# ============================================================== CA
def ca_gpu(n, state, steps, strategy, rho, world=1):
    maps = [tri.tri_map_init(n, rho, 1, g, world, 1) for g in range(world)]
    full = torch.from_numpy(state).cuda()
    cur = [full[mp.out_offset: mp.out_offset + mp.out_cells].clone() for mp in maps]
    nxt = [torch.empty_like(c) for c in cur]
    def row_of(r):   # halo row r as a copy from the rank that owns it (None if outside)
        for h, p in enumerate(maps):
            if p.row_begin <= r < p.row_end:
                o = T(r) - p.out_offset
                return cur[h][o: o + r + 1].clone()
        return None

    for _ in range(steps):
        for g, mp in enumerate(maps):
            above = row_of(mp.row_begin - 1) if mp.row_begin > 0 else None
            below = row_of(mp.row_end) if mp.row_end < n else None
            if mp.out_cells:
                tri.tri_ca_step(mp, strategy, cur[g], nxt[g], above, below)
        sync()
        cur, nxt = nxt, cur
    return np.concatenate([c.cpu().numpy() for c in cur])


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("rho", [128, 224, 256, 512])
@pytest.mark.parametrize("n,seed,steps", [(1, 7, 2), (2, 42, 3), (3, 7, 2), (17, 42, 5), (130, 7, 6),
                                          (1000, 42, 4), (2049, 7, 3)])
def test_ca_small(orc, strategy, rho, n, seed, steps):
    st = inputs.ca_state(n, seed)
    assert np.array_equal(ca_gpu(n, st, steps, strategy, rho), orc.ca_run(n, st, steps))


@pytest.mark.parametrize("world", [2, 3, 7])
def test_ca_ranks_with_halos(orc, world):
    n = 1500
    st = inputs.ca_state(n, 42)
    assert np.array_equal(ca_gpu(n, st, 5, "lambda", 128, world), orc.ca_run(n, st, 5))


@pytest.mark.parametrize("rho", [128, 224, 256, 512])
@pytest.mark.parametrize("n", [1000, 2049])
def test_ca_ignores_bytes_past_the_slice(orc, rho, n):
    """State buffers embedded in 0xFF-filled allocations: whatever lies past the
    packed slice (or past a row) must never leak into a cell."""
    D = T(n)
    st = inputs.ca_state(n, 7)
    bigA = torch.full((D + 4096,), 255, dtype=torch.uint8, device="cuda")
    bigB = torch.full((D + 4096,), 255, dtype=torch.uint8, device="cuda")
    a, b = bigA[:D], bigB[:D]
    a.copy_(torch.from_numpy(st))
    m = tri.tri_map_init(n, rho)
    for _ in range(3):
        tri.tri_ca_step(m, "lambda", a, b)
        a, b = b, a
    sync()
    assert np.array_equal(a.cpu().numpy(), orc.ca_run(n, st, 3))
    assert (bigA[D:] == 255).all() and (bigB[D:] == 255).all()     # nothing written past the slice


def ca_steps_gpu(n, state, calls, k, strategy, world=1, fill=None, rho=128):
    """`calls` launches of tri_ca_steps(k) per rank, ranks emulated on one GPU with
    deep halos (k packed rows from the owning rank)."""
    maps = [tri.tri_map_init(n, rho, 1, g, world, 1) for g in range(world)]
    full = torch.from_numpy(state).cuda()

    def buf(c):
        if fill is None:
            return torch.empty(max(c, 16), dtype=torch.uint8, device="cuda")
        return torch.full((c + 4096,), fill, dtype=torch.uint8, device="cuda")[:max(c, 16)]

    cur = []
    for mp in maps:
        b = buf(mp.out_cells)
        b[:mp.out_cells].copy_(full[mp.out_offset: mp.out_offset + mp.out_cells])
        cur.append(b)
    nxt = [buf(mp.out_cells) for mp in maps]

    def rows(r_lo, r_hi):   # packed rows [r_lo, r_hi) copied from their owners
        out = []
        for h, p in enumerate(maps):
            a, b = max(r_lo, p.row_begin), min(r_hi, p.row_end)
            if a < b:
                out.append(cur[h][T(a) - p.out_offset: T(b) - p.out_offset])
        return torch.cat(out).clone() if out else None

    for _ in range(calls):
        for g, mp in enumerate(maps):
            if not mp.out_cells:
                continue
            above = rows(max(mp.row_begin - k, 0), mp.row_begin) if mp.row_begin > 0 else None
            below = rows(mp.row_end, min(mp.row_end + k, n)) if mp.row_end < n else None
            tri.tri_ca_steps(mp, strategy, k, cur[g], nxt[g], above, below)
        sync()
        cur, nxt = nxt, cur
    return np.concatenate([c[:mp.out_cells].cpu().numpy() for c, mp in zip(cur, maps)])


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("k", [1, 2, 3, 5, 8, 9, 12, 16])
@pytest.mark.parametrize("n,seed", [(1, 7), (2, 42), (17, 7), (130, 42), (1000, 7), (2049, 42)])
def test_ca_steps_single(orc, strategy, k, n, seed):
    st = inputs.ca_state(n, seed)
    assert np.array_equal(ca_steps_gpu(n, st, 2, k, strategy), orc.ca_run(n, st, 2 * k))


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("k", [1, 2, 3, 5, 7, 8])
@pytest.mark.parametrize("n,seed", [(1, 7), (2, 42), (17, 7), (225, 42), (1000, 7), (2049, 42)])
def test_ca_steps_rho224(orc, strategy, k, n, seed):
    """The rho = 224 geometry (two words per phase-B thread, 256-column bitmaps)."""
    st = inputs.ca_state(n, seed)
    assert np.array_equal(ca_steps_gpu(n, st, 2, k, strategy, rho=224), orc.ca_run(n, st, 2 * k))


# ---- tri_ca_run: the bit-packed state (pack once, 8 generations per launch, unpack once)
@pytest.mark.parametrize("strategy", ["lambda", "bb", "persist"])
@pytest.mark.parametrize("n,seed,steps", [(1, 7, 3), (2, 42, 1), (31, 7, 9), (33, 42, 4), (224, 7, 8),
                                          (225, 42, 17), (700, 7, 0), (700, 42, 1), (1000, 7, 13),
                                          (2049, 42, 25), (4000, 7, 16)])
def test_ca_run_packed(orc, strategy, n, seed, steps):
    st = inputs.ca_state(n, seed)
    m = tri.tri_map_init(n, 240)
    x = torch.from_numpy(st).cuda()
    y = torch.full_like(x, 0x77)
    tri.tri_ca_run(m, strategy, steps, x, y)
    sync()
    assert np.array_equal(y.cpu().numpy(), orc.ca_run(n, st, steps))
    assert np.array_equal(x.cpu().numpy(), st)                   # the input is not modified


def test_ca_run_packed_patterns_and_alias(orc):
    """Glider, blinker, the diagonal L-triomino (still only because the cell that would
    complete it is outside the triangle) on the packed state; input and output aliased."""
    n = 300
    st = np.zeros(T(n), np.uint8)
    def put(i, j):
        st[T(i) + j] = 1
    for (i, j) in ((150, 40), (151, 41), (152, 39), (152, 40), (152, 41)):    # glider
        put(i, j)
    for (i, j) in ((200, 10), (200, 11), (200, 12)):                           # blinker
        put(i, j)
    for (i, j) in ((100, 100), (101, 100), (101, 101)):                        # L-triomino
        put(i, j)
    x = torch.from_numpy(st).cuda()
    m = tri.tri_map_init(n, 240)
    tri.tri_ca_run(m, "lambda", 20, x, x)
    sync()
    assert np.array_equal(x.cpu().numpy(), orc.ca_run(n, st, 20))


@pytest.mark.parametrize("world,k,rho", [(2, 4, 224), (3, 8, 224), (4, 3, 224)])
def test_ca_steps_deep_halo_ranks_rho224(orc, world, k, rho):
    n = 2000
    st = inputs.ca_state(n, 42)
    assert np.array_equal(ca_steps_gpu(n, st, 3, k, "lambda", world, rho=rho), orc.ca_run(n, st, 3 * k))


@pytest.mark.parametrize("k", [1, 8])
def test_ca_steps_ignores_garbage_rho224(orc, k):
    n = 2049
    st = inputs.ca_state(n, 7)
    assert np.array_equal(ca_steps_gpu(n, st, 2, k, "lambda", 1, fill=255, rho=224), orc.ca_run(n, st, 2 * k))


@pytest.mark.parametrize("world,k", [(2, 4), (3, 3), (4, 8), (3, 1), (2, 16), (3, 11)])
def test_ca_steps_deep_halo_ranks(orc, world, k):
    n = 2000
    st = inputs.ca_state(n, 42)
    assert np.array_equal(ca_steps_gpu(n, st, 3, k, "lambda", world), orc.ca_run(n, st, 3 * k))


@pytest.mark.parametrize("k", [1, 4, 16])
def test_ca_steps_ignores_garbage(orc, k):
    n = 2049
    st = inputs.ca_state(n, 7)
    assert np.array_equal(ca_steps_gpu(n, st, 2, k, "lambda", 1, fill=255), orc.ca_run(n, st, 2 * k))


@pytest.mark.parametrize("k,rho", [(4, 128), (8, 128), (16, 128), (8, 224)])
def test_ca_steps_full_size_sampled(orc, k, rho):
    """BASELINE configs[3] (n = 32768) with k-generation launches (the bench's plan uses
    the k it measures fastest), sampled rows."""
    n = 32768
    st = inputs.ca_state(n, 42)
    m = tri.tri_map_init(n, rho)
    a = torch.from_numpy(st).cuda()
    b = torch.empty_like(a)
    tri.tri_ca_steps(m, "lambda", k, a, b)
    sync()
    got = b.cpu().numpy()
    ref = st
    for _ in range(k):
        ref = orc.ca_step(n, ref)
    for rb, re in [(0, 40), (16380, 16390), (32700, 32768)]:
        assert np.array_equal(got[T(rb):T(re)], ref[T(rb):T(re)])


@pytest.mark.slow
def test_large_n_64bit_offsets(orc):
    """n = 200000: 2.0e10 packed cells (> 2^32) -- EDM (80 GB) and one CA generation
    (2 x 20 GB) through the 64-bit index paths, sampled rows vs the oracle."""
    n = 200000
    D = T(n)
    assert D > 2**34
    pts = inputs.points(n, 3, 7)
    m = tri.tri_map_init(n, 128)
    out = torch.empty(D, dtype=torch.float32, device="cuda")
    tri.tri_edm(m, "lambda", torch.from_numpy(pts).cuda(), out)
    sync()
    for rb, re in [(0, 8), (92681, 92684), (199997, 200000)]:        # T(92681) crosses 2^32
        edm_close(out[T(rb):T(re)].cpu().numpy(), orc.edm(pts, rb, re))
    del out
    torch.cuda.empty_cache()
    # CA just past 2^32 cells (n = 92800: 4.31e9 bytes); Bernoulli(0.5) bits from a
    # seeded numpy generator (the torch generator would need 17 GB of host floats)
    n = 92800
    D = T(n)
    assert D > 2**32
    st = np.random.default_rng(7).integers(0, 2, size=D, dtype=np.uint8)
    m = tri.tri_map_init(n, 128)
    a = torch.from_numpy(st).cuda()
    b = torch.empty_like(a)
    tri.tri_ca_step(m, "lambda", a, b)
    sync()
    for rb, re in [(92680, 92683), (92797, 92800)]:                  # T(92681) crosses 2^32
        assert np.array_equal(b[T(rb):T(re)].cpu().numpy(), orc.ca_step_rows(n, st, rb, re))
    tri.tri_ca_steps(m, "lambda", 3, a, b)
    sync()
    for rb, re in [(92680, 92683), (92790, 92800)]:
        lo, hi = rb - 3, min(re + 3, n)          # light cone: 3 generations of rows [lo, hi)
        work = np.zeros(D, np.uint8)            # are exact on [rb, re)
        work[T(lo):T(hi)] = st[T(lo):T(hi)]
        for _ in range(3):
            nxt = np.zeros(D, np.uint8)
            nxt[T(lo):T(hi)] = orc.ca_step_rows(n, work, lo, hi)
            work = nxt
        assert np.array_equal(b[T(rb):T(re)].cpu().numpy(), work[T(rb):T(re)])
    del a, b
    torch.cuda.empty_cache()


def test_ca_100_steps(orc):
    n = 2048
    st = inputs.ca_state(n, 7)
    assert np.array_equal(ca_gpu(n, st, 100, "persist", 512), orc.ca_run(n, st, 100))


def test_ca_full_size_sampled_rows(orc):
    """BASELINE configs[3]: n = 32768; 2 generations, sampled row bands vs the oracle."""
    n = 32768
    st = inputs.ca_state(n, 42)
    m = tri.tri_map_init(n, 512)
    a = torch.from_numpy(st).cuda()
    b = torch.empty_like(a)
    prev = st
    for _ in range(2):
        tri.tri_ca_step(m, "persist", a, b)
        sync()
        got = b.cpu().numpy()
        for rb, re in [(0, 40), (10000, 10010), (32700, 32768)]:
            assert np.array_equal(got[T(rb):T(re)], orc.ca_step_rows(n, prev, rb, re))
        prev = got
        a, b = b, a


# ============================================================== triplet
def triplet_close(got, ref, scale):
    err = np.abs(got - ref)
    assert np.all(err <= 1e-5 * scale + 1e-300), (float((err / scale).max()))


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("rho", [8, 16, 32])
@pytest.mark.parametrize("n,seed,gen", [(3, 7, "lattice"), (4, 42, "lattice"), (17, 7, "points"),
                                        (40, 42, "lattice"), (100, 7, "points"), (300, 42, "lattice")])
def test_triplet_small(orc, strategy, rho, n, seed, gen):
    x = inputs.lattice4(n, seed) if gen == "lattice" else inputs.points4(n, seed)
    tm = tri.tet_map_init(n, rho)
    e = torch.empty(n, dtype=torch.float64, device="cuda")
    tri.tet_triplet(tm, strategy, torch.from_numpy(x).cuda(), e, nu=1.0)
    sync()
    got = e.cpu().numpy()
    ref, A = orc.triplet(x), orc.triplet_abs(x)
    triplet_close(got, ref, A)
    assert abs(got.sum() - ref.sum()) <= 1e-5 * A.sum()


@pytest.mark.parametrize("rho", [8, 32])
def test_triplet_ranks_and_nu(orc, rho):
    n = 200
    x = inputs.points4(n, 7)
    d = torch.from_numpy(x).cuda()
    tot = np.zeros(n)
    for g in range(4):
        tm = tri.tet_map_init(n, rho, g, 4)
        e = torch.empty(n, dtype=torch.float64, device="cuda")
        tri.tet_triplet(tm, "persist", d, e, nu=2.5)
        sync()
        tot += e.cpu().numpy()
    triplet_close(tot, orc.triplet(x, nu=2.5), orc.triplet_abs(x, nu=2.5))


def test_triplet_full_size_sampled(orc):
    """BASELINE configs[4]: n = 4096, fp32 points; sampled particles vs the oracle."""
    n = 4096
    x = inputs.points4(n, 42)
    tm = tri.tet_map_init(n, 32)
    e = torch.empty(n, dtype=torch.float64, device="cuda")
    tri.tet_triplet(tm, "persist", torch.from_numpy(x).cuda(), e)
    sync()
    got = e.cpu().numpy()
    for t0 in (0, 2047, 4090):
        t1 = t0 + 4 if t0 < 4090 else 4096
        triplet_close(got[t0:t1], orc.triplet(x, 1.0, t0, t1), orc.triplet_abs(x, 1.0, t0, t1))


# ============================================================== ABI errors on device
def test_abi_rejects_bad_buffers():
    m = tri.tri_map_init(100, 128)
    small = torch.empty(10, dtype=torch.float32, device="cuda")
    pts = torch.rand(100, 3, device="cuda")
    with pytest.raises(tri.TriError) as e:
        tri.tri_edm(m, "lambda", pts, small)
    assert e.value.code == tri.TRI_EINVAL
    with pytest.raises(tri.TriError):
        tri.tri_edm(tri.tri_map_init(100, 16), "lambda", pts, torch.empty(T(100), device="cuda"))
    with pytest.raises(tri.TriError):
        tri.tri_dummy(tri.tri_map_init(100, 64), "lambda", tri.TRI_DUMMY_DIGEST,
                      torch.zeros(1, dtype=torch.int64, device="cuda"))


# ============================================================== 1-D collision (Eq. 5 tiles)
@pytest.mark.parametrize("strategy", ["lambda", "bb"])
@pytest.mark.parametrize("n,seed,rmax", [(1, 7, 0.1), (2, 42, 0.9), (255, 7, 0.01), (256, 42, 0.01),
                                         (1000, 7, 0.003), (5000, 42, 2e-4), (70001, 7, 1e-5)])
def test_collide1d(orc, strategy, n, seed, rmax):
    iv = inputs.intervals(n, seed, rmax)
    m = tri.tri_map_init(n, 256)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_collide1d(m, strategy, torch.from_numpy(iv).cuda(), cnt)
    sync()
    assert cnt.item() == orc.collide1d(iv)


def test_collide1d_ranks_and_quantized(orc):
    n = 30000
    iv = inputs.intervals(n, 42, 1e-4, bits=20)
    d = torch.from_numpy(iv).cuda()
    for strategy in ("lambda", "bb"):
        tot = 0
        for g in range(3):
            m = tri.tri_map_init(n, 256, 1, g, 3, 1)
            cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
            tri.tri_collide1d(m, strategy, d, cnt)
            sync()
            tot += cnt.item()
        assert tot == orc.collide1d(iv)


@pytest.mark.parametrize("offset,scale", [(0.0, 1.0), (100.0, 1.0), (-3000.0, 10.0), (0.0, 1e-4)])
def test_collide1d_knife_edge_pairs(orc, offset, scale):
    """The 1-D hot loop only filters on widened end points; partners placed at
    |ci - cj| = (ri + rj)(1 + delta), delta within a few ulps, must be counted exactly."""
    rng = np.random.default_rng(3)
    h = 4096
    c = rng.random(h) * scale + offset
    r = rng.random(h) * 1e-3 * scale
    rp = rng.random(h) * 1e-3 * scale
    sign = np.where(rng.random(h) < 0.5, -1.0, 1.0)
    delta = rng.integers(-8, 9, size=h) * 2.0 ** -24
    iv = np.zeros((2 * h, 2), np.float32)
    iv[:h, 0], iv[:h, 1] = c, r
    iv[h:, 0], iv[h:, 1] = c + sign * (r + rp) * (1 + delta), rp
    ref = orc.collide1d(iv)
    assert ref > 100
    d = torch.from_numpy(iv).cuda()
    for strategy in ("lambda", "bb"):
        m = tri.tri_map_init(len(iv), 256)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        tri.tri_collide1d(m, strategy, d, cnt)
        sync()
        assert cnt.item() == ref, strategy


# ============================================================== succinct LUT tetrahedral map
@pytest.mark.parametrize("shift", [0, 4, 9, 40])
def test_tet_lut_map_matches_enumeration(orc, shift):
    """Layer index from the succinct table (S = T3, G = bucket starts) + 2-D lambda:
    identical to the triple-loop enumeration, every Eq. / successor check passes."""
    I, J, K = orc.enumerate_tet(120)
    kmax, cnt = 119, len(I) - 1                 # omega + 1 is mapped too: stay below T3(120)
    lut = torch.empty(tri.tet_lut_bytes(kmax, shift), dtype=torch.uint8, device="cuda")
    tri.tet_lut_build(kmax, shift, lut)
    ijk = torch.empty(3 * cnt, dtype=torch.int32, device="cuda")
    fail = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tet_map_eval_lut(0, cnt, kmax, shift, lut, ijk, fail)
    sync()
    got = ijk.cpu().numpy().astype(np.uint32).reshape(-1, 3)
    assert np.array_equal(got[:, 0], I[:cnt]) and np.array_equal(got[:, 1], J[:cnt])
    assert np.array_equal(got[:, 2], K[:cnt])
    assert fail.item() == 0


@pytest.mark.parametrize("kmax,shift,w0,count", [(511, 13, 0, None), (4000, 20, None, 1 << 24)])
def test_tet_lut_map_equals_cbrt_map(kmax, shift, w0, count):
    """n = 4096 at rho = 8 (512 layers, every omega) and a 4001-layer table near its end:
    the table map and the cube-root map give the same (i, j, k)."""
    end = (kmax + 1) * (kmax + 2) * (kmax + 3) // 6
    if count is None:
        count = end - 1
    if w0 is None:
        w0 = end - 1 - count
    lut = torch.empty(tri.tet_lut_bytes(kmax, shift), dtype=torch.uint8, device="cuda")
    tri.tet_lut_build(kmax, shift, lut)
    a = torch.empty(3 * count, dtype=torch.int32, device="cuda")
    b = torch.empty_like(a)
    fa = torch.zeros(1, dtype=torch.int64, device="cuda")
    fb = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tet_map_eval_lut(w0, count, kmax, shift, lut, a, fa)
    tri.tet_map_eval(w0, count, b, fb)
    sync()
    assert fa.item() == 0 and fb.item() == 0
    assert torch.equal(a, b)
    with pytest.raises(tri.TriError) as e:                 # omega + 1 past the table
        tri.tet_map_eval_lut(end - 1, 1, kmax, shift, lut, None, fa)
    assert e.value.code == tri.TRI_ERANGE


# --------------------------------------------------------------------------- fused P2P halos
def _p2p_link(halos, bounds, n):
    from paper_1609_01490_b200 import dist as tdist
    for g, h in enumerate(halos):
        R0, R1 = bounds[g]
        if R1 <= R0:
            continue
        up = tdist.owner(bounds, R0 - 1) if R0 > 0 else None
        down = tdist.owner(bounds, R1) if R1 < n else None
        h.link([t.data_ptr() for t in halos[up].below] if up is not None else None,
               [t.data_ptr() for t in halos[down].above] if down is not None else None)


def ca_steps_p2p_gpu(n, state, calls, k, strategy, world, rho):
    """tri_ca_steps_p2p with ranks emulated on one GPU: every launch stores its first
    / last k rows straight into the neighbours' (parity-double-buffered) halo
    buffers; no exchange step between launches."""
    from paper_1609_01490_b200 import dist as tdist
    maps = [tri.tri_map_init(n, rho, 1, g, world, 1) for g in range(world)]
    bounds = [(m.row_begin, m.row_end) for m in maps]
    halos = [tdist.P2PHalo(bounds, n, g, k, exchange=False) for g in range(world)]
    _p2p_link(halos, bounds, n)
    full = torch.from_numpy(state).cuda()
    cur = [full[m.out_offset:m.out_offset + m.out_cells].clone() if m.out_cells else
           torch.empty(16, dtype=torch.uint8, device="cuda") for m in maps]
    nxt = [torch.empty_like(c) for c in cur]
    for g, (h, m) in enumerate(zip(halos, maps)):           # parity-0 halos = the initial state's rows
        R0, R1 = bounds[g]
        if R1 > R0 and R0 > 0:
            h.above[0][:h.na].copy_(full[T(max(R0 - k, 0)):T(R0)])
        if R1 > R0 and R1 < n:
            h.below[0][:h.nb].copy_(full[T(R1):T(min(R1 + k, n))])
    for e in range(calls):
        for g, m in enumerate(maps):
            if m.out_cells:
                tri.tri_ca_steps_p2p(m, strategy, k, cur[g], nxt[g], *halos[g].args(e))
        cur, nxt = nxt, cur
    sync()
    return np.concatenate([c[:m.out_cells].cpu().numpy() for c, m in zip(cur, maps)])


@pytest.mark.parametrize("world,k,rho", [(2, 1, 128), (2, 4, 128), (3, 8, 128), (4, 16, 128), (3, 3, 224),
                                         (2, 8, 224), (4, 5, 224)])
def test_ca_steps_p2p_emulated(orc, world, k, rho):
    n = 2000
    st = inputs.ca_state(n, 7)
    assert np.array_equal(ca_steps_p2p_gpu(n, st, 3, k, "lambda", world, rho), orc.ca_run(n, st, 3 * k))


@pytest.mark.parametrize("strategy", ["bb", "persist"])
@pytest.mark.parametrize("world,k,rho", [(3, 8, 224), (2, 5, 128)])
def test_ca_steps_p2p_strategies(orc, strategy, world, k, rho):
    """The peer stores live in the shared store phase: BB and the persistent walk too."""
    n = 1777
    st = inputs.ca_state(n, 42)
    assert np.array_equal(ca_steps_p2p_gpu(n, st, 2, k, strategy, world, rho), orc.ca_run(n, st, 2 * k))


def test_ca_steps_p2p_single_rank_is_tri_ca_steps(orc):
    """world = 1: no peers, the result equals tri_ca_steps."""
    n = 1000
    st = inputs.ca_state(n, 42)
    assert np.array_equal(ca_steps_p2p_gpu(n, st, 2, 8, "lambda", 1, 224), orc.ca_run(n, st, 16))


def _p2p_worker(rank, world, port, n, k, rho, calls, q):
    import os
    import torch.distributed as dist
    from paper_1609_01490_b200 import dist as tdist
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        maps = [tri.tri_map_init(n, rho, 1, g, world, 1) for g in range(world)]
        bounds = [(m.row_begin, m.row_end) for m in maps]
        m = maps[rank]
        st = inputs.ca_state(n, 7)
        cur = torch.from_numpy(st[m.out_offset:m.out_offset + m.out_cells].copy()).cuda()
        nxt = torch.empty_like(cur)
        h = tdist.P2PHalo(bounds, n, rank, k)          # CUDA IPC: maps the neighbour's buffers
        h.prime(cur)
        for e in range(calls):
            tri.tri_ca_steps_p2p(m, "lambda", k, cur, nxt, *h.args(e))
            h.epoch_barrier()
            cur, nxt = nxt, cur
        torch.cuda.synchronize()
        q.put((rank, cur.cpu().numpy()))
        dist.barrier()
        h.close()
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover - reported to the parent
        q.put((rank, repr(ex)))


@pytest.mark.parametrize("k,rho", [(4, 128), (8, 224)])
def test_ca_steps_p2p_two_processes_ipc(orc, k, rho):
    """Two processes (one GPU here, one per GPU in production) exchange CUDA IPC
    handles of their halo buffers; the kernels store into each other's memory."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n, world, calls = 1500, 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_p2p_worker, args=(g, world, port, n, k, rho, calls, q)) for g in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for g in range(world):
        assert not isinstance(got[g], str), got[g]
    st = inputs.ca_state(n, 7)
    assert np.array_equal(np.concatenate([got[g] for g in range(world)]), orc.ca_run(n, st, calls * k))
