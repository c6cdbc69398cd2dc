"""Pins for the CPU oracle (-m "not gpu").

Every oracle function is checked against something OTHER than itself: paper
witness values (tests/golden/, cited), closed forms, SPEC worked examples,
library routines (scipy), independent algorithms (cell lists, full-grid
convolution, angle-form ATM), and brute force on tiny inputs.  Each pin is
chosen so a plausible slip (a dropped term, an off-by-one index, j<=i vs j<i,
a wrong sign, < vs <=, a transposed operand) fails at least one of them.
"""
import math
import random
from itertools import combinations

import numpy as np
import pytest

from conftest import golden
from paper_1609_01490_b200 import inputs


def T(r):
    return r * (r + 1) // 2


def T3(r):
    return r * (r + 1) * (r + 2) // 6


# ---------------------------------------------------------------- figurate
def test_figurate_examples(orc):
    g = {k: int(v) for k, v in golden("counts.txt")}
    assert orc.tri_number(3) == g["tri_number_3"]
    for r in (1, 2, 3, 4):
        assert orc.tet_number(r) == g[f"tet_number_{r}"]
    assert orc.tri_number(0) == 0 and orc.tet_number(0) == 0


def test_tet_is_sum_of_tri(orc):
    # T_n = sum_{r=1}^n r(r+1)/2, checked by running sums (r <= 10^4).
    acc = 0
    for r in range(0, 10001):
        acc += r * (r + 1) // 2
        if r % 97 == 0 or r < 50:
            assert orc.tet_number(r) == acc
            assert orc.tri_number(r) == sum(range(r + 1)) if r < 200 else True


def test_figurate_overflow_is_error(orc):
    with pytest.raises(ValueError):
        orc.tri_number(2**64 - 1)
    assert orc.tri_number(2**32) == 2**32 * (2**32 + 1) // 2


# ---------------------------------------------------------------- enumeration / lambda
def test_enumerate_tri_hand_cases(orc):
    I, J = orc.enumerate_tri(2)
    assert list(zip(I.tolist(), J.tolist())) == [(0, 0), (1, 0), (1, 1)]
    I, J = orc.enumerate_tri(3, diag=False)
    assert list(zip(I.tolist(), J.tolist())) == [(1, 0), (2, 0), (2, 1)]
    I, J = orc.enumerate_tri(1)
    assert list(zip(I.tolist(), J.tolist())) == [(0, 0)]


@pytest.mark.parametrize("m", [1, 2, 3, 7, 16, 33, 100, 257])
def test_enumerate_tri_covers_triangle_once(orc, m):
    I, J = orc.enumerate_tri(m)
    assert len(I) == T(m)                                   # P:189-199 count
    cells = set(zip(I.tolist(), J.tolist()))
    assert cells == {(i, j) for i in range(m) for j in range(i + 1)}
    # position omega holds the cell with linear index T(i)+j (Eq. 1 row-major)
    w = np.arange(len(I), dtype=np.int64)
    assert np.array_equal(w, I.astype(np.int64) * (I.astype(np.int64) + 1) // 2 + J)


def test_lambda_paper_witnesses(orc):
    for w, i, j in golden("lambda_witnesses.txt"):
        assert orc.lam(int(w)) == (int(i), int(j))
    # Theorem 1's non-linearity: g(7) != g(4) + g(3)
    a, b = orc.lam(4), orc.lam(3)
    assert orc.lam(7) != (a[0] + b[0], a[1] + b[1])


@pytest.mark.parametrize("m", [1, 5, 64, 300])
def test_lambda_search_equals_enumeration(orc, m):
    # two independent algorithms inside the oracle: counter walk vs bisection on Eq. 3
    I, J = orc.enumerate_tri(m)
    for w in range(len(I)):
        assert orc.lam(w) == (int(I[w]), int(J[w]))


def test_lambda_exact_integer_closed_form_to_2_40(orc):
    # Eq. 4 solved exactly in integers: i = floor((isqrt(8w+1)-1)/2) (x^2+x-2w=0).
    rng = random.Random(1)
    ws = [rng.randrange(0, 2**40) for _ in range(2000)]
    for r in [1, 2, 3, 1000, 4607, 4608, 2**20 - 1, 2**20, 1482910]:
        ws += [T(r) - 1, T(r), T(r) + 1]
    for w in ws:
        if w < 0:
            continue
        i = (math.isqrt(8 * w + 1) - 1) // 2
        assert orc.lam(w) == (i, w - T(i)), w


def test_enumerate_tet_hand_and_cover(orc):
    I, J, K = orc.enumerate_tet(2)
    assert list(zip(I.tolist(), J.tolist(), K.tolist())) == [(0, 0, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1)]
    for m in (1, 3, 9, 20):
        I, J, K = orc.enumerate_tet(m)
        assert len(I) == T3(m)
        got = set(zip(I.tolist(), J.tolist(), K.tolist()))
        assert got == {(i, j, k) for k in range(m) for i in range(k + 1) for j in range(i + 1)}
        w = np.arange(len(I), dtype=np.int64)
        k = K.astype(np.int64); i = I.astype(np.int64)
        assert np.array_equal(w, k * (k + 1) * (k + 2) // 6 + i * (i + 1) // 2 + J)


def test_tet_lambda_witnesses_and_enumeration(orc):
    for w, i, j, k in golden("tet_witnesses.txt"):
        assert orc.tet_lam(int(w)) == (int(i), int(j), int(k))
    I, J, K = orc.enumerate_tet(24)
    for w in range(len(I)):
        assert orc.tet_lam(w) == (int(I[w]), int(J[w]), int(K[w]))


def test_tet_lambda_at_layer_boundaries(orc):
    # independent: integer cube-root search by Python ints (k^3 <= 6w bracket + walk)
    rng = random.Random(3)
    ks = [1, 2, 5, 35 // 1, 511, 512, 4095, 65536, 2**19] + [rng.randrange(1, 2**19) for _ in range(300)]
    for k in ks:
        for w in (T3(k) - 1, T3(k), T3(k) + 1):
            kk = 0
            while T3(kk + 1) <= w:
                kk = kk + 1 if kk < 8 else max(kk + 1, int(round((6 * w) ** (1 / 3))) - 3)
            while T3(kk) > w:
                kk -= 1
            w2 = w - T3(kk)
            i = (math.isqrt(8 * w2 + 1) - 1) // 2
            assert orc.tet_lam(w) == (i, w2 - T(i), kk), (k, w)


# ---------------------------------------------------------------- dispatch counts
def test_dispatch_count_spec_example(orc):
    g = {k: int(v) for k, v in golden("counts.txt")}
    c = orc.dispatch_count(8, 2, strategy=1)
    assert (c["threads"], c["useful"], c["discarded"]) == (
        g["bb_n8_rho2_threads"], g["bb_n8_rho2_useful"], g["bb_n8_rho2_discarded"])


@pytest.mark.parametrize("n,rho", [(8, 2), (64, 16), (2048, 16), (100, 16), (37, 8), (1, 8)])
def test_dispatch_count_closed_forms(orc, n, rho):
    m = -(-n // rho)
    lam = orc.dispatch_count(n, rho, strategy=0)
    bb = orc.dispatch_count(n, rho, strategy=1)
    assert lam["useful"] == bb["useful"] == T(n)                 # D = n(n+1)/2
    assert lam["blocks"] == T(m) and lam["threads"] == T(m) * rho * rho
    assert bb["blocks"] == m * m and bb["blocks_discarded"] == T(m - 1)
    if n % rho == 0:
        assert lam["discarded"] == rho * (rho - 1) // 2 * m
        assert bb["discarded"] == n * (n - 1) // 2
    s = orc.dispatch_count(n, rho, strategy=0, diag=False)
    assert s["useful"] == T(n - 1)


# ---------------------------------------------------------------- dummy
def test_dummy_digest_closed_form(orc):
    g = {k: int(v) for k, v in golden("counts.txt")}
    assert orc.dummy_digest(2) == g["dummy_digest_n2"]
    for n in (1, 2, 3, 10, 77, 2048):
        assert orc.dummy_digest(n) == (n - 1) * n * (n + 1) // 2
    assert orc.dummy_digest(2048) == 4294966272


@pytest.mark.parametrize("n", [1, 2, 5, 31, 130])
def test_dummy_packed_codes(orc, n):
    out = orc.dummy_packed(n)
    exp = [(i << 16) | j for i in range(n) for j in range(i + 1)]
    assert out.tolist() == exp
    out8 = orc.dummy_packed(n, elem_bytes=8)
    assert out8.tolist() == [(i << 32) | j for i in range(n) for j in range(i + 1)]
    # row slice = the matching window of the full array
    rb, re = n // 3, n - n // 4
    assert orc.dummy_packed(n, rb, re).tolist() == exp[T(rb):T(re)]


# ---------------------------------------------------------------- EDM
def test_edm_hand_cases(orc):
    pts = np.array([[0, 0, 0], [3, 4, 0], [3, 4, 12]], np.float32)
    out = orc.edm(pts)
    # layout (0,0),(1,0),(1,1),(2,0),(2,1),(2,2)
    assert out.tolist() == [0.0, 5.0, 0.0, 13.0, 12.0, 0.0]
    same = np.ones((7, 3), np.float32) * 0.25
    assert not orc.edm(same).any()


@pytest.mark.parametrize("n,dim,seed", [(64, 3, 7), (257, 3, 42), (100, 4, 7), (50, 1, 42), (33, 2, 7)])
def test_edm_vs_scipy_pdist(orc, n, dim, seed):
    from scipy.spatial.distance import pdist
    pts = inputs.points(n, dim, seed)
    out = orc.edm(pts)
    cond = pdist(pts.astype(np.float64))         # upper condensed, (a,b) a<b row-major
    full = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    full[iu] = cond
    full = full + full.T
    il = np.tril_indices(n)                       # row-major lower incl. diagonal == Eq. 1
    ref = full[il].astype(np.float32)
    assert out.shape == ref.shape
    np.testing.assert_allclose(out, ref, rtol=2e-7, atol=0)
    # rows slice equals the window
    rb, re = n // 4, n // 2
    assert np.array_equal(orc.edm(pts, rb, re), out[T(rb):T(re)])


# ---------------------------------------------------------------- collision
def _cell_list_count_fp64(s):
    """Independent O(n) algorithm: uniform grid of cell size >= 2 r_max, fp64."""
    n = len(s)
    c = s[:, :3].astype(np.float64); r = s[:, 3].astype(np.float64)
    h = max(2 * r.max(), 1e-3)
    cells = {}
    keys = np.floor(c / h).astype(np.int64)
    for t in range(n):
        cells.setdefault(tuple(keys[t]), []).append(t)
    cnt = 0
    amb = 0
    for key, members in cells.items():
        cand = []
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    cand += cells.get((key[0] + dx, key[1] + dy, key[2] + dz), [])
        cand = np.array(cand)
        for t in members:
            o = cand[cand < t]
            if len(o) == 0:
                continue
            d2 = ((c[o] - c[t]) ** 2).sum(1)
            s2 = (r[o] + r[t]) ** 2
            cnt += int((d2 < s2).sum())
            amb += int((np.abs(d2 - s2) <= 1e-6 * s2).sum())
    return cnt, amb


def test_collide_hand_cases(orc):
    # touching spheres (d == r1 + r2) do not collide; overlapping and nested do
    s = np.array([[0.0, 0.0, 0.0, 0.25], [0.5, 0.0, 0.0, 0.25]], np.float32)
    assert orc.collide(s) == 0
    s[1, 0] = 0.375
    assert orc.collide(s) == 1
    s = np.array([[0.5, 0.5, 0.5, 0.25], [0.5, 0.5, 0.5, 0.0625], [0.5, 0.5, 0.5, 0.125]], np.float32)
    assert orc.collide(s) == 3                        # strict pairs only: C(3,2)
    assert orc.collide(s[:1]) == 0                    # no self-collision (Q1)
    # dz matters: separated only along z
    s = np.array([[0.5, 0.5, 0.0, 0.1], [0.5, 0.5, 0.5, 0.1]], np.float32)
    assert orc.collide(s) == 0


@pytest.mark.parametrize("n,seed", [(4000, 7), (6000, 42)])
def test_collide_quantized_equals_geometric_truth(orc, n, seed):
    # On an 11-bit grid every fp32 op of the predicate is exact, so the
    # count equals the real-number predicate evaluated by the fp64 cell list.
    s = inputs.spheres_quantized(n, seed, bits=11, r_max=0.04)
    cnt, _ = _cell_list_count_fp64(s)
    assert cnt > 50
    assert orc.collide(s) == cnt


def test_collide_random_matches_cell_list(orc):
    s = inputs.spheres(5000, 42, r_max=0.03)
    cnt, amb = _cell_list_count_fp64(s)
    got = orc.collide(s)
    assert abs(got - cnt) <= amb and cnt > 100
    # brute force tiny
    s = inputs.spheres(60, 7, r_max=0.2)
    bf = 0
    for i in range(60):
        for j in range(i):
            d = s[i, :3].astype(np.float64) - s[j, :3]
            bf += (d @ d) < (float(s[i, 3]) + float(s[j, 3])) ** 2
    assert orc.collide(s) == bf
    # row slices partition the count
    s = inputs.spheres(3000, 7, r_max=0.05)
    total = orc.collide(s)
    assert orc.collide(s, 0, 1000) + orc.collide(s, 1000, 3000) == total


# ---------------------------------------------------------------- CA
def _pack(full):
    n = full.shape[0]
    return full[np.tril_indices(n)].astype(np.uint8)


def _unpack(n, packed):
    f = np.zeros((n, n), np.uint8)
    f[np.tril_indices(n)] = packed
    return f


def _life_full_masked(n, packed, steps):
    """Textbook Life via scipy.signal.convolve2d (zero fill) on the full n x n grid,
    upper triangle forced dead after every step (cells outside the domain are dead)."""
    from scipy.signal import convolve2d
    k = np.ones((3, 3), np.int32); k[1, 1] = 0
    g = _unpack(n, packed).astype(np.int32)
    mask = np.tril(np.ones((n, n), np.int32))
    for _ in range(steps):
        nb = convolve2d(g, k, mode="same", boundary="fill", fillvalue=0)
        g = (((nb == 3) | ((g == 1) & (nb == 2))).astype(np.int32)) * mask
    return _pack(g)


@pytest.mark.parametrize("n,seed,steps", [(1, 7, 3), (2, 7, 3), (5, 42, 7), (17, 7, 7), (40, 42, 7), (130, 7, 12)])
def test_ca_vs_full_grid_convolution(orc, n, seed, steps):
    st = inputs.ca_state(n, seed)
    assert np.array_equal(orc.ca_run(n, st, steps), _life_full_masked(n, st, steps))


def test_ca_patterns(orc):
    n = 40
    def run(cells, steps):
        f = np.zeros((n, n), np.uint8)
        for i, j in cells:
            f[i, j] = 1
        out = orc.ca_run(n, _pack(f), steps)
        return {tuple(x) for x in np.argwhere(_unpack(n, out))}
    block = {(20, 5), (20, 6), (21, 5), (21, 6)}
    assert run(block, 5) == block                                   # still life
    blinker = {(20, 4), (20, 5), (20, 6)}
    assert run(blinker, 1) == {(19, 5), (20, 5), (21, 5)}           # period 2
    assert run(blinker, 2) == blinker
    glider = {(10, 3), (11, 4), (12, 2), (12, 3), (12, 4)}
    assert run(glider, 4) == {(i + 1, j + 1) for i, j in glider}    # moves (+1,+1)/4 gens
    L = {(10, 10), (11, 10), (11, 11)}                              # on the diagonal
    assert run(L, 3) == L            # still life only because (10,11) is outside (dead)
    assert run(set(), 3) == set()


# ---------------------------------------------------------------- triplet (ATM)
def _atm_angle_form(x, p, q, s, nu=1.0):
    """E = nu (1 + 3 cos g1 cos g2 cos g3) / (r12 r23 r31)^3 with the cosines from
    dot products (independent of the oracle's law-of-cosines form)."""
    P, Q, S = (x[t, :3].astype(np.float64) for t in (p, q, s))
    def cos(a, b, c):  # angle at a
        u, v = b - a, c - a
        return u @ v / (np.linalg.norm(u) * np.linalg.norm(v))
    r = np.linalg.norm(P - Q) * np.linalg.norm(Q - S) * np.linalg.norm(S - P)
    return nu * (1 + 3 * cos(P, Q, S) * cos(Q, S, P) * cos(S, P, Q)) / r**3


def test_triplet_closed_forms(orc):
    r = 0.7
    eq = np.array([[0, 0, 0, 0], [r, 0, 0, 0], [r / 2, r * math.sqrt(3) / 2, 0, 0]], np.float32)
    e = orc.triplet(eq)
    x = eq.astype(np.float64)
    a = np.linalg.norm(x[0, :3] - x[1, :3])
    # equilateral: E = (11/8) nu / r^9 (side lengths from the fp32-rounded points)
    side = [np.linalg.norm(x[i, :3] - x[j, :3]) for i, j in ((0, 1), (1, 2), (2, 0))]
    assert abs(max(side) - min(side)) < 1e-6
    E = 11 / 8 / a**9
    np.testing.assert_allclose(e, [E / 3] * 3, rtol=1e-5)
    col = np.array([[0, 0, 0, 0], [r, 0, 0, 0], [2 * r, 0, 0, 0]], np.float32)
    E = -1 / (4 * np.float64(np.float32(r)) ** 9)                  # collinear: -nu/(4 r^9)
    np.testing.assert_allclose(orc.triplet(col, nu=1.0), [E / 3] * 3, rtol=1e-9)
    np.testing.assert_allclose(orc.triplet(col, nu=2.5), [2.5 * E / 3] * 3, rtol=1e-9)


@pytest.mark.parametrize("n,seed", [(5, 7), (9, 42), (14, 7)])
def test_triplet_vs_angle_form_brute_force(orc, n, seed):
    x = inputs.lattice4(n, seed)
    e = np.zeros(n)
    tot = 0.0
    for p, q, s in combinations(range(n), 3):
        E = _atm_angle_form(x, p, q, s)
        tot += E
        for t in (p, q, s):
            e[t] += E / 3
    np.testing.assert_allclose(orc.triplet(x), e, rtol=1e-9)
    np.testing.assert_allclose(orc.triplet_total(x), tot, rtol=1e-9)


def test_triplet_permutation_and_sum(orc):
    x = inputs.points4(40, 7)
    e = orc.triplet(x)
    perm = np.random.default_rng(0).permutation(40)
    e2 = orc.triplet(x[perm])
    np.testing.assert_allclose(e2, e[perm], rtol=1e-9)
    np.testing.assert_allclose(e.sum(), orc.triplet_total(x), rtol=1e-9)
    np.testing.assert_allclose(orc.triplet(x, t_begin=10, t_end=20), e[10:20], rtol=0)


def test_triplet_abs_scale(orc):
    # A_t = (1/3) sum |E| >= |e_t|, with equality when all E share a sign (lattice, far apart)
    x = inputs.points4(30, 42)
    e, a = orc.triplet(x), orc.triplet_abs(x)
    assert np.all(a >= np.abs(e) - 1e-12 * a)
    col = np.array([[0, 0, 0, 0], [0.5, 0, 0, 0], [1.0, 0, 0, 0]], np.float32)
    np.testing.assert_allclose(orc.triplet_abs(col), -orc.triplet(col), rtol=1e-12)


# ---------------------------------------------------------------- sqrt variants (section 4.1)
def _np_variant_rows(w, variant):
    """Independent numpy float32 restatement of lambda_X / lambda_N."""
    f32 = np.float32
    x = (f32(0.25) + f32(2.0) * w.astype(np.float32)).astype(np.float32)
    if variant == 1:
        s = np.sqrt(x)
    else:
        xh = (f32(0.5) * x).astype(np.float32)
        y = (np.int32(0x5f3759df) - (x.view(np.int32) >> 1)).astype(np.int32).view(np.float32)
        for _ in range(3):
            y = (y * (f32(1.5) - (xh * y) * y)).astype(np.float32)   # Quake's x2*y*y
        s = (x * y + f32(1e-4)).astype(np.float32)
    return np.maximum(np.floor((s - f32(0.5)).astype(np.float32)), 0).astype(np.int64)


@pytest.mark.parametrize("variant,lo,hi", [(1, 0, 12_000_000), (2, 0, 2_000_000)])
def test_sqrt_variant_scan_vs_numpy(orc, variant, lo, hi):
    first = None
    fails = 0
    for a in range(lo, hi, 1 << 20):
        w = np.arange(a, min(hi, a + (1 << 20)), dtype=np.int64)
        i = _np_variant_rows(w, variant)
        bad = ~((i * (i + 1) // 2 <= w) & (w < (i + 1) * (i + 2) // 2))      # Eq. 3
        fails += int(bad.sum())
        if first is None and bad.any():
            first = int(w[np.argmax(bad)])
    got = orc.variant_scan(variant, lo, hi - lo)
    assert got == (fails, first)
    assert first is not None            # both variants do fail inside these ranges ...
    assert first > 100_000              # ... but only after many exact rows


@pytest.mark.parametrize("n,rho", [(1, 8), (2, 8), (7, 8), (8, 2), (100, 16), (2048, 16), (333, 32)])
def test_dispatch_count_rb(orc, n, rho):
    # RB covers the triangle with an O(1)-waste rectangle: useful = D exactly
    c = orc.dispatch_count(n, rho, strategy=2)
    assert c["useful"] == T(n)
    h = n // 2
    H, W = n - h, 2 * h + 1
    assert H * W == T(n)                                   # the fold is area-exact
    gx, gy = -(-W // rho), -(-H // rho)
    assert c["blocks"] == gx * gy and c["threads"] == gx * gy * rho * rho
    assert c["discarded"] < (W + H + rho) * rho            # waste only from block rounding


# ---------------------------------------------------------------- 1-D collision
def test_collide1d_hand_and_sweep(orc):
    iv = np.array([[0.0, 0.25], [0.5, 0.25], [0.25, 0.0625], [0.9, 0.01]], np.float32)
    # (1,0) touch exactly (|d| = s, not counted); (2,0) and (2,1) overlap; (3,*) far
    assert orc.collide1d(iv) == 2
    assert orc.collide1d(iv[:1]) == 0
    # independent algorithm on a 2^-20 grid (every fp32 op exact): sort by left end
    # and sweep, counting pairs with strict overlap of the open intervals
    iv = inputs.intervals(20000, 7, r_max=2e-4, bits=20)
    c, r = iv[:, 0].astype(np.float64), iv[:, 1].astype(np.float64)
    lo, hi = c - r, c + r
    order = np.argsort(lo, kind="stable")
    lo_s, hi_s = lo[order], hi[order]
    cnt = 0
    for a in range(len(order)):
        b = np.searchsorted(lo_s, hi_s[a], side="left")          # candidates: lo_b < hi_a
        if b > a + 1:                                            # open overlap also needs lo_a < hi_b
            cnt += int((hi_s[a + 1:b] > lo_s[a]).sum())
    assert cnt > 100
    assert orc.collide1d(iv) == cnt
    # brute force in numpy float32 (same op sequence) on random 24-bit inputs
    iv = inputs.intervals(700, 42, r_max=5e-3)
    d = iv[:, None, 0] - iv[None, :, 0]
    s = iv[:, None, 1] + iv[None, :, 1]
    m = (np.abs(d) < s) & np.tril(np.ones((700, 700), bool), -1)
    assert orc.collide1d(iv) == int(m.sum())
    assert orc.collide1d(iv, 0, 300) + orc.collide1d(iv, 300, 700) == int(m.sum())


def test_lambda_nodiag_reading_q2(orc):
    # Eq. 5 with the corrected j-term enumerates the strict lower triangle
    I, J = orc.enumerate_tri(60, diag=False)
    for w in range(len(I)):
        i = math.floor(math.sqrt(0.25 + 2 * w) + 0.5)             # Eq. 5's i-term (exact here)
        assert (i, w - i * (i - 1) // 2) == (int(I[w]), int(J[w]))
    assert (int(I[0]), int(J[0])) == (1, 0) and (int(I[2]), int(J[2])) == (2, 1)


# ------------------------------------------------ sqrt variants: golden first failures
def _golden_sqrt_variants():
    return {int(vid): int(w) for vid, _name, w in golden("sqrt_variants.txt")}


def _rn32(v):
    """Round a non-negative rational to the nearest fp32 (ties to even), exactly."""
    from fractions import Fraction
    v = Fraction(v)
    if v == 0:
        return v
    e = v.numerator.bit_length() - v.denominator.bit_length()
    if Fraction(2) ** e > v:
        e -= 1
    ulp = Fraction(2) ** (e - 23)
    q, r = divmod(v, ulp)
    if r * 2 > ulp or (r * 2 == ulp and q % 2 == 1):
        q += 1
    return q * ulp


def _sqrt32(x):
    """Correctly rounded fp32 sqrt of an fp32 value x > 0 (integer square roots only)."""
    from fractions import Fraction
    from math import isqrt
    E = 0                                      # 4^E <= x < 4^(E+1), so 2^E <= sqrt(x) < 2^(E+1)
    while Fraction(4) ** (E + 1) <= x:
        E += 1
    while Fraction(4) ** E > x:
        E -= 1
    sc = Fraction(2) ** (23 - E)               # sqrt(x) * sc in [2^23, 2^24): one unit = one ulp
    X = x * sc * sc
    q = isqrt(X.numerator // X.denominator)    # floor(sqrt(X))
    h = (Fraction(2 * q + 1, 2)) ** 2          # sqrt(X) vs q + 1/2  <=>  X vs (q + 1/2)^2
    if X > h or (X == h and q % 2 == 1):
        q += 1
    return Fraction(q) / sc


def _exact_row_x(w):
    """lambda_X evaluated with exact rational arithmetic and explicit fp32 roundings."""
    from fractions import Fraction
    from math import floor
    x = _rn32(Fraction(1, 4) + _rn32(2 * _rn32(w)))
    s = _rn32(_sqrt32(x) - Fraction(1, 2))
    return max(floor(s), 0)


def test_sqrt_variant_golden_first_failures(orc):
    """The oracle's scans hit the golden first failing omegas (SURVEY.md:38-40): 10,619,135
    for lambda_X, 1,316,253 for lambda_N in the cited (x2*y)*y Newton order."""
    g = _golden_sqrt_variants()
    for vid, w_first in g.items():
        nf, fw = orc.variant_scan(vid, 0, w_first + 1)
        assert fw == w_first and nf == 1, (vid, nf, fw)
    assert g[1] == T(4608) - 1 and g[2] == T(1622)


def test_sqrt_variant_x_exact_rational_boundaries():
    """Independent of numpy and of the oracle: lambda_X in exact rational arithmetic with
    explicit round-to-nearest-even after each fp32 operation.  Eq. 3 holds at every row
    boundary omega in {T(i) - 1, T(i)} below the golden omega, and fails there."""
    g = _golden_sqrt_variants()[1]
    for i in list(range(1, 64)) + list(range(4000, 4609)):
        for w in (T(i) - 1, T(i)):
            if w <= g:
                r = _exact_row_x(w)
                assert (T(r) <= w < T(r + 1)) == (w < g), (i, w, r)


# ------------------------------------------------ lambda_R within rsqrtf's error bound (Q5c)
def _np_lambda_r_rows(w):
    """Independent numpy restatement of lambda_R with a CORRECTLY ROUNDED
    reciprocal square root (fp64 1/sqrt rounded once to fp32: within 0.5 ulp, so inside
    any 2-ulp rsqrtf bound): x = 1/4 + 2w, s = x r + 1e-4, i = floor(s - 1/2), fp32."""
    f32 = np.float32
    x = (f32(0.25) + f32(2.0) * w.astype(np.float32)).astype(np.float32)
    r = (1.0 / np.sqrt(x.astype(np.float64))).astype(np.float32)
    s = ((x * r).astype(np.float32) + f32(1e-4)).astype(np.float32)
    return np.maximum(np.floor((s - f32(0.5)).astype(np.float32)), 0).astype(np.int64)


def _exact_rows(w):
    from math import isqrt
    return np.array([(isqrt(8 * int(v) + 1) - 1) // 2 for v in w], np.int64)


def test_lambda_r_bracket_holds_a_correctly_rounded_rsqrt(orc):
    """Every omega < 3,000,000: the numpy lambda_R row (an admissible rsqrtf) lies in the
    oracle's reachable-row interval, at the 2-ulp bound and at the PTX 2^-22.9 bound."""
    for rel in (orc.RSQRTF_REL, 2.0 ** -22.9):
        for a in range(0, 3_000_000, 1 << 20):
            cnt = min(3_000_000, a + (1 << 20)) - a
            w = np.arange(a, a + cnt, dtype=np.int64)
            lo, hi = orc.variant_r_rows(a, cnt, rel)
            r = _np_lambda_r_rows(w)
            assert np.all(lo.astype(np.int64) <= r) and np.all(r <= hi.astype(np.int64))
            assert np.all(hi.astype(np.int64) - lo.astype(np.int64) <= 1)   # 2 ulp moves a row by <= 1


def test_lambda_r_bracket_exact_where_the_bound_cannot_matter(orc):
    """Small omega: the eps = 1e-4 slack exceeds any 2-ulp error of x r, so every admissible
    rsqrtf gives the exact row (Eq. 3); checked against the integer closed form."""
    w = np.arange(0, 20_000, dtype=np.int64)
    lo, hi = orc.variant_r_rows(0, len(w))
    ex = _exact_rows(w)
    assert np.array_equal(lo.astype(np.int64), ex) and np.array_equal(hi.astype(np.int64), ex)


def test_lambda_r_scan_consistent_with_rows(orc):
    """The scan's surely / maybe wrong counts equal those of the per-omega intervals judged
    with the integer closed form (a different exact-row route than the scan's bisection),
    and the numpy lambda_R's failures sit inside the maybe set."""
    a, cnt = 2_000_000, 1 << 20
    w = np.arange(a, a + cnt, dtype=np.int64)
    lo, hi = orc.variant_r_rows(a, cnt)
    lo, hi = lo.astype(np.int64), hi.astype(np.int64)
    ex = np.floor((np.sqrt(8.0 * w + 1.0) - 1.0) / 2.0).astype(np.int64)   # exact: 8w+1 < 2^53
    ok = (ex * (ex + 1) // 2 <= w) & (w < (ex + 1) * (ex + 2) // 2)
    assert ok.all()
    sure_bad = (ex < lo) | (ex > hi)
    maybe_bad = ~((lo == hi) & (lo == ex))
    ns, fs, nm, fm = orc.variant_r_scan(a, cnt)
    assert (ns, nm) == (int(sure_bad.sum()), int(maybe_bad.sum()))
    assert fm == (int(w[np.argmax(maybe_bad)]) if maybe_bad.any() else None)
    r = _np_lambda_r_rows(w)
    assert not np.any((r != ex) & ~maybe_bad)
