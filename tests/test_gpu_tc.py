"""GPU tests of the tensor-core collision filter (-m gpu): the hardware accumulation
bound its margin assumes, and exact counts on inputs built to defeat a filter
(csrc/collide_tc.cu header; reading Q9)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1609_01490_b200 import inputs  # noqa: E402
from paper_1609_01490_b200 import tri  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    tri.lib()


def tf32(a):
    """Truncate fp32 values to TF32 (low 13 mantissa bits cleared): exact TF32 operands."""
    a = np.ascontiguousarray(a, np.float32)
    return (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def probe(X, Y):
    d = torch.empty((128, 128), dtype=torch.float32, device="cuda")
    tri.tri_tc_tf32_probe(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), d)
    torch.cuda.synchronize()
    return d.cpu().numpy().astype(np.float64)


def exact(X, Y):
    """Exact X Y^T: TF32 x TF32 products have <= 22 significant bits and the 8-term sums
    of these operands stay far inside fp64's 53 bits (checked by the exponent span)."""
    Xd, Yd = X.astype(np.float64), Y.astype(np.float64)
    terms = Xd[:, None, :] * Yd[None, :, :]
    return terms.sum(-1), np.abs(terms).sum(-1)


def cancelling_operands(seed, scale, jitter):
    """Rows x_i and columns y_j = x_i' + tiny, in the filter's form
    X = (x, P_hi, P_lo, 1, 1, 0), Y = (-2y, 1, 1, Q_hi, Q_lo, 0) with P = |x|^2, Q = |y|^2:
    X.Y = |x - y|^2 (+ split residue), the largest cancellation the filter meets."""
    rng = np.random.default_rng(seed)
    x = tf32(rng.uniform(-scale, scale, (128, 3)))
    y = tf32(x[rng.permutation(128)] + rng.normal(0, jitter * scale, (128, 3)))
    y[:64] = x[:64]                                   # and some exactly coincident pairs
    X = np.zeros((128, 8), np.float32)
    Y = np.zeros((128, 8), np.float32)
    P = (x.astype(np.float64) ** 2).sum(1)
    Q = (y.astype(np.float64) ** 2).sum(1)
    Ph = tf32(P.astype(np.float32)); Pl = tf32((P - Ph).astype(np.float32))
    Qh = tf32(Q.astype(np.float32)); Ql = tf32((Q - Qh).astype(np.float32))
    X[:, :3], X[:, 3], X[:, 4], X[:, 5], X[:, 6] = x, Ph, Pl, 1, 1
    Y[:, :3], Y[:, 3], Y[:, 4], Y[:, 5], Y[:, 6] = tf32(-2 * y), 1, 1, Qh, Ql
    return tf32(X), tf32(Y)


@pytest.mark.parametrize("case", ["random", "cancel_unit", "cancel_large", "cancel_tiny", "mixed_exponents"])
def test_tc_tf32_accumulation_bound(case):
    """The filter's margin assumes |fp32 tensor-core sum - exact sum| <= 2^-20 sum |x_k y_k|
    for one K = 8 tf32 MMA into a zeroed accumulator (csrc/collide_tc.cu).  Measured here
    on random and on maximally cancelling operands; the observed worst case is reported."""
    rng = np.random.default_rng(3)
    if case == "random":
        X, Y = tf32(rng.uniform(-1, 1, (128, 8))), tf32(rng.uniform(-1, 1, (128, 8)))
    elif case == "cancel_unit":
        X, Y = cancelling_operands(5, 0.5, 1e-3)
    elif case == "cancel_large":
        X, Y = cancelling_operands(6, 1000.0, 1e-6)
    elif case == "cancel_tiny":
        X, Y = cancelling_operands(7, 1e-3, 1e-2)
    else:
        e = rng.integers(-20, 20, (128, 8))
        X = tf32(rng.uniform(1, 2, (128, 8)) * np.exp2(e) * rng.choice([-1, 1], (128, 8)))
        Y = tf32(rng.uniform(1, 2, (128, 8)) * np.exp2(-e[rng.permutation(128)]) * rng.choice([-1, 1], (128, 8)))
    d = probe(X, Y)
    ex, ab = exact(X, Y)
    err = np.abs(d - ex)
    ratio = float((err / np.maximum(ab, 1e-300)).max())
    print(f"{case}: max |err| / sum|terms| = {ratio:.3e} (bound 2^-20 = {2.0 ** -20:.3e})")
    assert np.all(err <= 2.0 ** -20 * ab), ratio


def f16(a):
    return np.asarray(a, np.float64).astype(np.float16)


@pytest.mark.parametrize("case", ["cancel_unit", "cancel_large", "cancel_tiny", "random", "filter_shape"])
def test_tc_f16_accumulator_rounding(case):
    """The filter's sign test reads an F16 accumulator: it assumes D = round_f16(wide sum)
    -- products exact, summed in >= fp32 precision (within 2^-20 sum |x_k y_k| of the exact
    sum), rounded once to nearest (overflow to +-inf).  Then D's sign is the exact sum's
    whenever |exact| > 2^-20 sum |terms| and the rounding does not reach zero."""
    rng = np.random.default_rng(11)
    A = np.zeros((128, 16)); B = np.zeros((128, 16))
    if case == "random":
        A, B = rng.uniform(-2, 2, (128, 16)), rng.uniform(-2, 2, (128, 16))
    else:
        sc = {"cancel_unit": 0.5, "cancel_large": 60.0, "cancel_tiny": 0.01, "filter_shape": 0.5}[case]
        x = f16(rng.uniform(-sc, sc, (128, 3))).astype(np.float64)
        y = f16(x[rng.permutation(128)] + rng.normal(0, 1e-3 * sc, (128, 3))).astype(np.float64)
        y[:64] = x[:64]
        P, Q = (x ** 2).sum(1), (y ** 2).sum(1)
        P1 = f16(P).astype(np.float64); P2 = f16((P - P1) * 2048).astype(np.float64)
        Q1 = f16(Q).astype(np.float64); Q2 = f16((Q - Q1) * 2048).astype(np.float64)
        S = 32768.0 if case == "filter_shape" else 1.0          # the filter's column scale
        A[:, :3], A[:, 3], A[:, 4], A[:, 5], A[:, 6] = x, P1, P2, 1, 1 / 2048
        B[:, :3], B[:, 3], B[:, 4], B[:, 5], B[:, 6] = -2 * S * y, S, S / 2048, S * Q1, S * Q2
    A, B = f16(A), f16(B)
    d = torch.empty((128, 128), dtype=torch.int16, device="cuda")
    tri.tri_tc_f16_probe(torch.from_numpy(A.view(np.int16)).cuda(), torch.from_numpy(B.view(np.int16)).cuda(), d)
    torch.cuda.synchronize()
    D = d.cpu().numpy().view(np.float16).astype(np.float64)
    Ad, Bd = A.astype(np.float64), B.astype(np.float64)
    ex = Ad @ Bd.T
    ab = (np.abs(Ad)[:, None, :] * np.abs(Bd)[None, :, :]).sum(-1)
    lo = f16(ex - 2.0 ** -20 * ab).astype(np.float64)            # round_f16 of the end points of
    hi = f16(ex + 2.0 ** -20 * ab).astype(np.float64)            # the wide sum's error interval
    assert np.all((D >= np.minimum(lo, hi)) & (D <= np.maximum(lo, hi)))
    sure = np.abs(ex) > 2.0 ** -20 * ab + 2.0 ** -24
    assert np.array_equal(np.signbit(D)[sure], (ex < 0)[sure])


@pytest.mark.parametrize("strategy,rho", [("tc", 384), ("bb_tc", 256), ("tc", 512), ("tc", 1024), ("bb_tc", 1024)])
def test_collide_tc_special_values(orc, strategy, rho):
    """NaN, infinite and huge coordinates or radii never break exactness: the filter
    treats them as never- or always-flagged and the exact predicate decides."""
    s = inputs.spheres(3000, 9, 0.05)
    s[10] = [np.nan, 0.5, 0.5, 0.01]
    s[20, 3] = np.nan
    s[30] = [np.inf, 0.2, 0.2, 0.01]
    s[40] = [1e20, 1e20, 0.0, 0.01]
    s[41] = [1e20, 1e20, 0.0, 0.01]                    # coincident with 40: counted in fp32
    s[50, 3] = 3.0                                     # a huge sphere overlapping most others
    s[2990] = s[5]                                     # an exactly coincident pair, far apart in index
    s[2991, :3] = s[6, :3]
    s[2991, 3] = 0.0                                   # zero radius inside a sphere
    m = tri.tri_map_init(len(s), rho)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_collide(m, strategy, torch.from_numpy(s).cuda(), cnt)
    torch.cuda.synchronize()
    assert cnt.item() == orc.collide(s)


@pytest.mark.parametrize("strategy", ["tc", "bb_tc"])
def test_collide_tc_dense_cluster(orc, strategy):
    """Every pair of a dense cluster collides (every group flagged, every column recounted):
    the count is C(n, 2) on the diagonal and off-diagonal tiles alike."""
    n = 1500
    rng = np.random.default_rng(4)
    s = np.zeros((n, 4), np.float32)
    s[:, :3] = 0.3 + rng.random((n, 3)) * 1e-3
    s[:, 3] = 0.01
    for rho in (384, 1024):
        m = tri.tri_map_init(n, rho)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        tri.tri_collide(m, strategy, torch.from_numpy(s).cuda(), cnt)
        torch.cuda.synchronize()
        assert cnt.item() == orc.collide(s) == n * (n - 1) // 2, rho
