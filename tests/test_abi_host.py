"""Host-side tests of the C ABI (-m "not gpu"): the library loads, exports every
symbol include/tri.h declares, and its pure-host entry points (descriptor,
partition, host mirror of lambda) agree with the oracle.  No kernel launches."""
import math
import os
import random
import re
import subprocess

import pytest

from conftest import ROOT

tri = pytest.importorskip("paper_1609_01490_b200.tri")


@pytest.fixture(scope="module")
def L():
    from paper_1609_01490_b200 import build
    build.build()
    return tri.lib()


def header_functions():
    src = open(os.path.join(ROOT, "include", "tri.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b((?:tri|tet)_\w+)\s*\(", src, re.M)))


def test_header_parses():
    fns = header_functions()
    for must in ("tri_map_init", "tri_dummy", "tri_edm", "tri_collide", "tri_ca_step", "tet_triplet",
                 "tri_tc_tf32_probe", "tri_tc_f16_probe", "tri_collide_workspace_size"):
        assert must in fns


def test_library_exports_every_header_symbol(L):
    out = subprocess.run(["nm", "-D", "--defined-only", tri.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT\s+(\w+)$", out, re.M))
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing
    for f in header_functions():
        assert hasattr(L, f)
    assert set(tri.SIGNATURES) == set(header_functions())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", tri.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def T(r):
    return r * (r + 1) // 2


def test_status_strings(L):
    assert tri.status_str(0) == "TRI_OK"
    assert "EINVAL" in tri.status_str(-1)


def test_map_init_single(L):
    m = tri.tri_map_init(2048, 16)
    assert (m.m, m.blocks, m.cells) == (128, 8256, 2098176)
    assert (m.omega_begin, m.omega_end, m.row_begin, m.row_end) == (0, 8256, 0, 2048)
    assert (m.out_offset, m.out_cells) == (0, 2098176)
    assert m.waste_lambda == 15360 and m.waste_bb == 2096128
    m = tri.tri_map_init(65536, 128)
    assert m.blocks == 512 * 513 // 2 and m.cells == 2147516416


@pytest.mark.parametrize("n,rho,world", [(65536, 16, 8), (65536, 128, 8), (1000, 32, 3), (37, 8, 4),
                                         (200000, 256, 8), (100, 128, 2), (5, 128, 4)])
def test_partition_snapped(L, n, rho, world):
    maps = [tri.tri_map_init(n, rho, 1, g, world, 1) for g in range(world)]
    m = -(-n // rho)
    B = T(m)
    # contiguous cover of [0, B) and of the packed slice [0, D)
    assert maps[0].omega_begin == 0 and maps[-1].omega_end == B
    assert maps[0].out_offset == 0 and maps[-1].out_offset + maps[-1].out_cells == T(n)
    for a, b in zip(maps, maps[1:]):
        assert a.omega_end == b.omega_begin and a.row_end == b.row_begin
        assert a.out_offset + a.out_cells == b.out_offset
    # snapped row R_g minimises |T(R) - g B / world|, ties to the smaller (reading Q17)
    R = [min(range(m + 1), key=lambda r: (abs(world * T(r) - g * B), r)) for g in range(world + 1)]
    for g, x in enumerate(maps):
        assert x.omega_begin == T(R[g]) and x.omega_end == T(R[g + 1])
        assert x.row_begin == min(R[g] * rho, n) and x.row_end == min(R[g + 1] * rho, n)
    maps = [x for x in maps if x.row_begin // rho < m]
    if n == 65536 and rho == 16 and world == 8:      # SURVEY §8a a1 (derived bounds)
        assert [x.row_begin // rho for x in maps] + [m] == [0, 1448, 2048, 2508, 2896, 3238, 3547, 3831, 4096]


@pytest.mark.parametrize("n,rho,world", [(200000, 256, 8), (1000, 64, 3), (10, 64, 4)])
def test_partition_plain(L, n, rho, world):
    maps = [tri.tri_map_init(n, rho, 1, g, world, 0) for g in range(world)]
    B = T(-(-n // rho))
    for g, x in enumerate(maps):
        assert x.omega_begin == g * B // world and x.omega_end == (g + 1) * B // world


def test_map_init_errors(L):
    for args in [(0, 16), (10, 0), (10, 2000), (10, 16, 1, 2, 2), (10, 16, 1, -1, 2)]:
        with pytest.raises(tri.TriError) as e:
            tri.tri_map_init(*args)
        assert e.value.code == tri.TRI_EINVAL
    with pytest.raises(tri.TriError) as e:
        tri.tri_map_init(2**31 + 1, 1)
    assert e.value.code == tri.TRI_ERANGE


@pytest.mark.parametrize("rho,k,ok", [(128, 16, True), (128, 17, False), (224, 8, True), (224, 9, False),
                                      (256, 1, False), (224, 0, False)])
def test_ca_steps_geometry_validation(L, rho, k, ok):
    """tri_ca_steps accepts (rho = 128, k <= 16) and (rho = 224, k <= 8) only; a bad
    pair returns EINVAL synchronously, before any launch (fake device pointers)."""
    import ctypes
    m = tri.tri_map_init(1000, rho)
    if ok:
        return      # a valid pair would launch: covered by the GPU tests
    big = m.out_cells
    rc = L.tri_ca_steps(ctypes.byref(m), 0, k, ctypes.c_void_p(1 << 20), big, ctypes.c_void_p(2 << 20), big,
                        None, 0, None, 0, None, None)
    assert rc == tri.TRI_EINVAL


def test_ca_steps_p2p_validation(L):
    """tri_ca_steps_p2p: misaligned peer pointers, a rank owning fewer than k rows and
    bad (rho, k) pairs are EINVAL before any launch (fake device pointers); the IPC
    calls reject NULLs."""
    import ctypes
    vp = ctypes.c_void_p
    A, B, P = vp(1 << 20), vp(2 << 20), vp(3 << 20)
    m = tri.tri_map_init(1000, 128, 1, 1, 2, 1)
    call = lambda mp, k, pa: L.tri_ca_steps_p2p(ctypes.byref(mp), 0, k, A, mp.out_cells, B, mp.out_cells,
                                                None, 0, None, 0, pa, None, None, None)
    assert call(m, 4, vp((3 << 20) + 8)) == tri.TRI_EINVAL          # peer not 16-byte aligned
    assert call(m, 17, P) == tri.TRI_EINVAL                         # k > 16 at rho = 128
    small = tri.tri_map_init(230, 224, 1, 1, 2, 1)                  # rank 1 owns rows [224, 230)
    assert (small.row_begin, small.row_end) == (224, 230)
    assert call(small, 8, P) == tri.TRI_EINVAL                      # owns 6 < k rows, sends to a peer
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64(0)
    assert L.tri_ipc_handle(None, h, ctypes.byref(off)) == tri.TRI_EINVAL
    p, b = vp(), vp()
    assert L.tri_ipc_open(None, 0, ctypes.byref(p), ctypes.byref(b)) == tri.TRI_EINVAL
    assert L.tri_ipc_close(None) == tri.TRI_EINVAL


@pytest.mark.parametrize("rho", [384, 640, 768, 1024])
def test_collide_rho384_is_tc_only(L, rho):
    """rho = 384, 640, ..., 1024 are tile edges of the tcgen05 collision kernel only: the
    SIMT strategies reject them with EINVAL before any launch (fake device pointers)."""
    import ctypes
    m = tri.tri_map_init(1000, rho)
    for strat in (tri.TRI_LAMBDA, tri.TRI_BB, tri.TRI_LAMBDA_PERSIST):
        assert L.tri_collide(ctypes.byref(m), strat, ctypes.c_void_p(1 << 20), 16 * 1000,
                             ctypes.c_void_p(2 << 20), 8, None, 0, None) == tri.TRI_EINVAL


def test_host_lambda_vs_oracle(L, orc):
    rng = random.Random(5)
    ws = list(range(0, 5000)) + [rng.randrange(0, 2**40) for _ in range(3000)]
    for r in (4607, 4608, 2**20, 1482909, 1482910):
        ws += [T(r) - 1, T(r), T(r) + 1]
    for w in ws:
        if w < 2**40:
            assert tri.tri_lambda(w) == orc.lam(w)
    with pytest.raises(tri.TriError):
        tri.tri_lambda(2**40)


def test_host_tet_lambda_vs_oracle(L, orc):
    rng = random.Random(6)
    ws = list(range(0, 3000)) + [rng.randrange(0, 2**40) for _ in range(2000)]
    for k in (5, 35, 511, 512, 4096, 10000):
        t3 = k * (k + 1) * (k + 2) // 6
        ws += [t3 - 1, t3, t3 + 1]
    for w in ws:
        assert tri.tet_lambda(w) == orc.tet_lam(w)


def test_tet_map_init(L):
    t = tri.tet_map_init(4096, 8)
    assert t.m == 512 and t.blocks == 512 * 513 * 514 // 6 == 22500864
    useful = 4096 * 4095 * 4094 // 6
    assert t.waste_tet == t.blocks * 512 - useful
    assert abs((t.waste_bb + useful) / (t.blocks * 512) - 5.965) < 1e-3    # ~6x
    t = tri.tet_map_init(4096, 16)
    assert t.blocks == 256 * 257 * 258 // 6
    parts = [tri.tet_map_init(4096, 16, g, 4) for g in range(4)]
    assert parts[0].omega_begin == 0 and parts[-1].omega_end == t.blocks
    for a, b in zip(parts, parts[1:]):
        assert a.omega_end == b.omega_begin
    with pytest.raises(tri.TriError):
        tri.tet_map_init(4096, 5)


def test_host_lambda_nodiag_vs_oracle(L, orc):
    I, J = orc.enumerate_tri(400, diag=False)
    for w in range(len(I)):
        assert tri.tri_lambda_nodiag(w) == (int(I[w]), int(J[w]))
    for w in (2**39, 2**40 - 1):
        i, j = tri.tri_lambda_nodiag(w)
        assert i * (i - 1) // 2 <= w < i * (i + 1) // 2 and j == w - i * (i - 1) // 2


def test_tet_lut_bytes(L):
    """Succinct layer table size: 8 (kmax + 2) + 4 (nb + 1), nb = (T3(kmax+1) >> shift) + 1."""
    def t3(k):
        return k * (k + 1) * (k + 2) // 6
    for kmax, shift in [(1, 0), (119, 4), (511, 13), (4000, 20), (2 ** 20 - 1, 40)]:
        nb = (t3(kmax + 1) >> shift) + 1
        assert tri.tet_lut_bytes(kmax, shift) == 8 * (kmax + 2) + 4 * (nb + 1)
    for kmax, shift in [(0, 5), (2 ** 20, 5), (10, -1), (10, 41)]:
        assert tri.tet_lut_bytes(kmax, shift) == 0
    # validation happens before any launch (no GPU needed): NULL buffer, short buffer
    assert L.tet_lut_build(511, 13, None, 0, None) == tri.TRI_EINVAL
    assert L.tet_lut_build(511, 13, 8, tri.tet_lut_bytes(511, 13) - 1, None) == tri.TRI_EINVAL
    assert L.tet_map_eval_lut(0, 10, 511, 13, None, None, 8, None) == tri.TRI_EINVAL


# ---------------------------------------------------------------- capacities (include/tri.h conventions)
def test_edm_host_validation(L):
    """tri_edm_host runs tri_edm's checks before touching any buffer: a tile edge outside
    {32, 64, 128, 256}, dim = 5, a short point workspace, a short band workspace, a
    short host output, the RB strategy and a bad map all return EINVAL (fake pointers:
    nothing is launched or copied)."""
    import ctypes
    vp = ctypes.c_void_p
    n = 1000
    H, D, O, W = vp(1 << 20), vp(1 << 24), vp(1 << 26), vp(1 << 28)

    def call(m, strat=0, dim=3, pts_ws=4 * 3 * n, out=None, ws=1 << 24, band=0, pts=4 * 3 * n):
        out = 4 * m.out_cells if out is None else out
        return L.tri_edm_host(ctypes.byref(m), strat, H, dim, dim, pts, D, pts_ws, O, out, W, ws, band)

    m16 = tri.tri_map_init(n, 16)
    assert call(m16) == tri.TRI_EINVAL                                   # rho = 16: no EDM kernel
    m = tri.tri_map_init(n, 128)
    assert call(m, dim=5, pts=4 * 5 * n, pts_ws=4 * 5 * n) == tri.TRI_EINVAL   # dim outside 1..4
    assert call(m, pts_ws=4 * 3 * n - 4) == tri.TRI_EINVAL               # point workspace one float short
    assert call(m, pts=4 * 3 * n - 4) == tri.TRI_EINVAL                  # host points one float short
    assert call(m, out=4 * m.out_cells - 1) == tri.TRI_EINVAL            # host output one byte short
    assert call(m, ws=2 * 4 * 1000) == tri.TRI_EINVAL                    # a tile row (<= 128 000 cells) > a half
    assert call(m, band=4096) == tri.TRI_EINVAL                          # ... or > band_cells
    assert call(m, strat=tri.TRI_RB) == tri.TRI_EINVAL                   # RB has no band form
    assert call(m, strat=99) == tri.TRI_EINVAL
    bad = tri.tri_map_init(n, 128)
    bad.m += 1                                                           # inconsistent descriptor
    assert call(bad) == tri.TRI_EINVAL
    ns = tri.tri_map_init(n, 128, 1, 0, 2, 0)                            # unsnapped multi-rank map
    assert call(ns) == tri.TRI_EINVAL


def test_edm_capacities(L):
    import ctypes
    vp = ctypes.c_void_p
    m = tri.tri_map_init(1000, 128)
    f = lambda pts, out, ld=3: L.tri_edm(ctypes.byref(m), 0, vp(1 << 20), 3, ld, pts, vp(1 << 24), out, None)
    assert f(4 * 3 * 1000 - 4, 4 * m.out_cells) == tri.TRI_EINVAL
    assert f(4 * 3 * 1000, 4 * m.out_cells - 4) == tri.TRI_EINVAL
    assert f(4 * 4 * 1000 - 8, 4 * m.out_cells, ld=4) == tri.TRI_EINVAL   # strided rows: (n-1) ld + dim floats
    m16 = tri.tri_map_init(1000, 16)
    assert L.tri_edm(ctypes.byref(m16), 0, vp(1 << 20), 3, 3, 12000, vp(1 << 24), 4 * m16.out_cells,
                     None) == tri.TRI_EINVAL


def test_collide_triplet_ca_capacities(L):
    """Short inputs / outputs are EINVAL before any launch (fake device pointers)."""
    import ctypes
    vp = ctypes.c_void_p
    n = 1000
    m = tri.tri_map_init(n, 256)
    c = lambda sb, cb, strat=0, cnt=vp(2 << 20): L.tri_collide(ctypes.byref(m), strat, vp(1 << 20), sb, cnt, cb,
                                                              None, 0, None)
    assert c(16 * n - 16, 8) == tri.TRI_EINVAL                  # one sphere short
    assert c(16 * n, 4) == tri.TRI_EINVAL                       # an int32 count
    assert c(16 * n, 8, cnt=vp((2 << 20) + 4)) == tri.TRI_EINVAL  # count not 8-byte aligned
    assert c(16 * n, 8, strat=tri.STRATEGIES["bb_tc"] + 1) == tri.TRI_EINVAL
    # the tensor-core strategies need their workspace: m * rho * 64 bytes
    mt = tri.tri_map_init(n, 384)
    need = L.tri_collide_workspace_size(ctypes.byref(mt), 8)
    assert need == 256 + mt.m * 384 * 64 and L.tri_collide_workspace_size(ctypes.byref(mt), 0) == 0
    for strat in (8, 9):
        assert L.tri_collide(ctypes.byref(mt), strat, vp(1 << 20), 16 * n, vp(2 << 20), 8, vp(3 << 20), need - 16,
                             None) == tri.TRI_EINVAL
        assert L.tri_collide(ctypes.byref(mt), strat, vp(1 << 20), 16 * n, vp(2 << 20), 8, None, need,
                             None) == tri.TRI_EINVAL
        assert L.tri_collide(ctypes.byref(mt), strat, vp(1 << 20), 16 * n, vp(2 << 20), 8, vp((3 << 20) + 8), need,
                             None) == tri.TRI_EINVAL
    assert L.tri_collide1d(ctypes.byref(m), 0, vp(1 << 20), 8 * n - 8, vp(2 << 20), 8, None) == tri.TRI_EINVAL
    assert L.tri_collide1d(ctypes.byref(m), 0, vp(1 << 20), 8 * n, vp(2 << 20), 4, None) == tri.TRI_EINVAL
    tm = tri.tet_map_init(64, 8)
    t = lambda pb, eb: L.tet_triplet(ctypes.byref(tm), 0, vp(1 << 20), pb, 1.0, vp(2 << 20), eb, None)
    assert t(16 * 63, 8 * 64) == tri.TRI_EINVAL
    assert t(16 * 64, 8 * 63) == tri.TRI_EINVAL
    mc = tri.tri_map_init(1000, 128, 1, 1, 2, 1)               # rank 1 of 2: both halos exist
    R0, R1 = mc.row_begin, mc.row_end
    assert R0 > 0 and R1 == 1000
    oc = mc.out_cells
    s1 = lambda ib, ob, ab: L.tri_ca_step(ctypes.byref(mc), 0, vp(1 << 20), ib, vp(1 << 24), ob, vp(1 << 26), ab,
                                          None, 0, None, None)
    assert s1(oc - 1, oc, R0) == tri.TRI_EINVAL
    assert s1(oc, oc - 1, R0) == tri.TRI_EINVAL
    assert s1(oc, oc, R0 - 1) == tri.TRI_EINVAL                 # the halo row above is R0 bytes
    k = 4
    sk = lambda ab: L.tri_ca_steps(ctypes.byref(mc), 0, k, vp(1 << 20), oc, vp(1 << 24), oc, vp(1 << 26), ab,
                                   None, 0, None, None)
    assert sk(T(R0) - T(R0 - k) - 1) == tri.TRI_EINVAL          # k rows above: T(R0) - T(R0 - k) bytes


def test_ca_run_validation(L):
    """tri_ca_run: world 1, rho 224, capacities, workspace, steps >= 0 -- EINVAL before any launch."""
    import ctypes
    vp = ctypes.c_void_p
    n = 1000
    m = tri.tri_map_init(n, 240)
    D = n * (n + 1) // 2
    ws = L.tri_ca_run_workspace_size(ctypes.byref(m))
    assert ws == 2 * (((D + 31) // 32 * 4 + 255) // 256 * 256)
    run = lambda mp, st=0, steps=5, ib=D, ob=D, wb=ws, w=vp(3 << 20): L.tri_ca_run(
        ctypes.byref(mp), st, steps, vp(1 << 20), ib, vp(2 << 20), ob, w, wb, None)
    assert run(m, ib=D - 1) == tri.TRI_EINVAL
    assert run(m, ob=D - 1) == tri.TRI_EINVAL
    assert run(m, wb=ws - 1) == tri.TRI_EINVAL
    assert run(m, w=None) == tri.TRI_EINVAL
    assert run(m, steps=-1) == tri.TRI_EINVAL
    assert run(m, st=tri.TRI_LAMBDA_CLC) == tri.TRI_EINVAL
    assert run(tri.tri_map_init(n, 224)) == tri.TRI_EINVAL                 # rho 240 only
    assert run(tri.tri_map_init(n, 240, 1, 0, 2, 1)) == tri.TRI_EINVAL     # one rank only


def test_map_rows_variant_validation(L):
    """tri_map_rows_variant: a bad variant, a NULL / misaligned pointer or a short capacity
    is EINVAL, an omega range past 2^40 ERANGE -- synchronously, before any launch."""
    import ctypes
    p = ctypes.c_void_p(1 << 20)
    assert L.tri_map_rows_variant(0, 0, 10, p, 40, None) == tri.TRI_EINVAL          # not a variant
    assert L.tri_map_rows_variant(4, 0, 10, p, 40, None) == tri.TRI_EINVAL
    assert L.tri_map_rows_variant(3, 0, 10, None, 40, None) == tri.TRI_EINVAL
    assert L.tri_map_rows_variant(3, 0, 10, ctypes.c_void_p((1 << 20) + 2), 40, None) == tri.TRI_EINVAL
    assert L.tri_map_rows_variant(3, 0, 10, p, 39, None) == tri.TRI_EINVAL           # 10 rows need 40 B
    assert L.tri_map_rows_variant(3, 1 << 40, 1, p, 4, None) == tri.TRI_ERANGE
