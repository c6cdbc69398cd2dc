"""CPU oracle for arXiv:1609.01490 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this package.  The product package
``paper_1609_01490_b200`` never imports it and shares no code with it.

Every result here is the plain definition (a double loop over j <= i < n,
fp64 unless the method fixes the precision), implemented in ``oracle.c`` and
marshalled through ctypes.  Citations are in ``oracle.c`` next to each
function ("P:a-b" = PAPER.md lines).  Parity status of every function is
"pinned" (tests/test_oracle_pins.py); nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

u64 = ctypes.c_uint64
i64 = ctypes.c_int64
i32 = ctypes.c_int32
vp = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, OpenMP, no fp contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.orc_tri_number.argtypes = [u64, ctypes.POINTER(u64)]
        L.orc_tet_number.argtypes = [u64, ctypes.POINTER(u64)]
        L.orc_enumerate_tri.argtypes = [i64, i32, vp, vp, u64]
        L.orc_enumerate_tri.restype = i64
        L.orc_enumerate_tet.argtypes = [i64, vp, vp, vp, u64]
        L.orc_enumerate_tet.restype = i64
        L.orc_lambda.argtypes = [u64, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]
        L.orc_tet_lambda.argtypes = [u64] + [ctypes.POINTER(ctypes.c_uint32)] * 3
        L.orc_dummy_packed.argtypes = [i64, i64, i64, vp, i32]
        L.orc_dummy_digest.argtypes = [i64]
        L.orc_dummy_digest.restype = u64
        L.orc_dispatch_count.argtypes = [i64, i32, i32, i32, vp]
        L.orc_edm.argtypes = [i64, vp, i32, i64, i64, i64, vp]
        L.orc_collide.argtypes = [i64, vp, i64, i64, ctypes.POINTER(u64)]
        L.orc_ca_step.argtypes = [i64, vp, vp]
        L.orc_ca_run.argtypes = [i64, vp, i64]
        L.orc_ca_step_rows.argtypes = [i64, vp, vp, i64, i64]
        L.orc_triplet.argtypes = [i64, vp, ctypes.c_double, i64, i64, vp]
        L.orc_triplet_abs.argtypes = [i64, vp, ctypes.c_double, i64, i64, vp]
        L.orc_triplet_total.argtypes = [i64, vp, ctypes.c_double, ctypes.POINTER(ctypes.c_double)]
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_set_threads.restype = None
        L.orc_variant_scan.argtypes = [i32, u64, u64, ctypes.POINTER(u64), ctypes.POINTER(u64)]
        L.orc_collide1d.argtypes = [i64, vp, i64, i64, ctypes.POINTER(u64)]
        L.orc_variant_r_rows.argtypes = [u64, u64, ctypes.c_double, vp, vp]
        L.orc_variant_r_scan.argtypes = [u64, u64, ctypes.c_double] + [ctypes.POINTER(u64)] * 4
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise ValueError(f"oracle error {rc}")


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_threads(k: int) -> None:
    """OpenMP threads of later oracle calls (k < 1: all cores)."""
    lib().orc_set_threads(int(k))


# --- figurate numbers ----------------------------------------------------
def tri_number(r: int) -> int:
    out = u64()
    _check(lib().orc_tri_number(r, ctypes.byref(out)))
    return out.value


def tet_number(r: int) -> int:
    out = u64()
    _check(lib().orc_tet_number(r, ctypes.byref(out)))
    return out.value


# --- enumerations (Eq. 1 / tetrahedral layers) ---------------------------
def enumerate_tri(m: int, diag: bool = True):
    cnt = m * (m + 1) // 2 if diag else max(m * (m - 1) // 2, 0)
    I = np.zeros(max(cnt, 1), np.uint32)
    J = np.zeros(max(cnt, 1), np.uint32)
    got = lib().orc_enumerate_tri(m, 1 if diag else 0, _ptr(I), _ptr(J), cnt)
    if got < 0:
        raise ValueError(got)
    return I[:got], J[:got]


def enumerate_tet(m: int):
    cnt = m * (m + 1) * (m + 2) // 6
    I = np.zeros(max(cnt, 1), np.uint32)
    J = np.zeros(max(cnt, 1), np.uint32)
    K = np.zeros(max(cnt, 1), np.uint32)
    got = lib().orc_enumerate_tet(m, _ptr(I), _ptr(J), _ptr(K), cnt)
    if got < 0:
        raise ValueError(got)
    return I[:got], J[:got], K[:got]


def lam(omega: int):
    bi, bj = ctypes.c_uint32(), ctypes.c_uint32()
    _check(lib().orc_lambda(omega, ctypes.byref(bi), ctypes.byref(bj)))
    return bi.value, bj.value


def tet_lam(omega: int):
    i, j, k = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
    _check(lib().orc_tet_lambda(omega, ctypes.byref(i), ctypes.byref(j), ctypes.byref(k)))
    return i.value, j.value, k.value


def variant_scan(variant: int, w0: int, count: int):
    """Section 4.1 sqrt variants (1 = lambda_X, 2 = lambda_N), uncorrected:
    (number of omega in [w0, w0+count) they get wrong, first such omega or None)."""
    f, first = u64(), u64()
    _check(lib().orc_variant_scan(variant, w0, count, ctypes.byref(f), ctypes.byref(first)))
    return f.value, (None if first.value == 2**64 - 1 else first.value)


RSQRTF_REL = 2.0 ** -22        # rsqrtf: 2 ulp (CUDA Math API) -- DESIGN.md reading Q5c


def variant_r_rows(w0: int, count: int, rel: float = RSQRTF_REL):
    """lambda_R within rsqrtf's error bound: per omega in [w0, w0+count) the
    lowest and highest row any fp32 r with |r sqrt(x) - 1| <= rel can give."""
    lo, hi = np.zeros(count, np.uint32), np.zeros(count, np.uint32)
    _check(lib().orc_variant_r_rows(w0, count, rel, _ptr(lo), _ptr(hi)))
    return lo, hi


def variant_r_scan(w0: int, count: int, rel: float = RSQRTF_REL):
    """(n surely wrong, first surely wrong, n maybe wrong, first maybe wrong) for lambda_R on
    [w0, w0+count): surely = the exact row is reachable by no admissible rsqrtf, maybe = by
    not every one.  first = None when there is none."""
    a, b, c, d = u64(), u64(), u64(), u64()
    _check(lib().orc_variant_r_scan(w0, count, rel, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                                    ctypes.byref(d)))
    nn = lambda v: None if v == 2**64 - 1 else v
    return a.value, nn(b.value), c.value, nn(d.value)


# --- dummy ----------------------------------------------------------------
def dummy_packed(n: int, row_begin: int = 0, row_end: int | None = None, elem_bytes: int = 4):
    row_end = n if row_end is None else row_end
    cnt = row_end * (row_end + 1) // 2 - row_begin * (row_begin + 1) // 2
    out = np.zeros(max(cnt, 1), np.uint32 if elem_bytes == 4 else np.uint64)
    _check(lib().orc_dummy_packed(n, row_begin, row_end, _ptr(out), elem_bytes))
    return out[:cnt]


def dummy_digest(n: int) -> int:
    return int(lib().orc_dummy_digest(n))


def dispatch_count(n: int, rho: int, strategy: int, diag: bool = True):
    c = np.zeros(5, np.uint64)
    _check(lib().orc_dispatch_count(n, rho, strategy, 1 if diag else 0, _ptr(c)))
    return dict(blocks=int(c[0]), blocks_discarded=int(c[1]), threads=int(c[2]),
                useful=int(c[3]), discarded=int(c[4]))


# --- EDM ------------------------------------------------------------------
def edm(pts: np.ndarray, row_begin: int = 0, row_end: int | None = None) -> np.ndarray:
    pts = np.ascontiguousarray(pts, np.float32)
    n, dim = pts.shape
    row_end = n if row_end is None else row_end
    cnt = row_end * (row_end + 1) // 2 - row_begin * (row_begin + 1) // 2
    out = np.zeros(max(cnt, 1), np.float32)
    _check(lib().orc_edm(n, _ptr(pts), dim, dim, row_begin, row_end, _ptr(out)))
    return out[:cnt]


# --- collision --------------------------------------------------------------
def collide(spheres: np.ndarray, row_begin: int = 0, row_end: int | None = None) -> int:
    s = np.ascontiguousarray(spheres, np.float32)
    assert s.ndim == 2 and s.shape[1] == 4
    n = s.shape[0]
    row_end = n if row_end is None else row_end
    out = u64()
    _check(lib().orc_collide(n, _ptr(s), row_begin, row_end, ctypes.byref(out)))
    return out.value


def collide1d(intervals: np.ndarray, row_begin: int = 0, row_end: int | None = None) -> int:
    s = np.ascontiguousarray(intervals, np.float32)
    assert s.ndim == 2 and s.shape[1] == 2
    n = s.shape[0]
    row_end = n if row_end is None else row_end
    out = u64()
    _check(lib().orc_collide1d(n, _ptr(s), row_begin, row_end, ctypes.byref(out)))
    return out.value


# --- CA -------------------------------------------------------------------
def ca_step(n: int, state: np.ndarray) -> np.ndarray:
    s = np.ascontiguousarray(state, np.uint8)
    out = np.zeros_like(s)
    _check(lib().orc_ca_step(n, _ptr(s), _ptr(out)))
    return out


def ca_run(n: int, state: np.ndarray, steps: int) -> np.ndarray:
    s = np.array(state, np.uint8, copy=True, order="C")
    _check(lib().orc_ca_run(n, _ptr(s), steps))
    return s


def ca_step_rows(n: int, state: np.ndarray, row_begin: int, row_end: int) -> np.ndarray:
    s = np.ascontiguousarray(state, np.uint8)
    cnt = row_end * (row_end + 1) // 2 - row_begin * (row_begin + 1) // 2
    out = np.zeros(max(cnt, 1), np.uint8)
    _check(lib().orc_ca_step_rows(n, _ptr(s), _ptr(out), row_begin, row_end))
    return out[:cnt]


# --- triplet ----------------------------------------------------------------
def triplet(pts4: np.ndarray, nu: float = 1.0, t_begin: int = 0, t_end: int | None = None) -> np.ndarray:
    p = np.ascontiguousarray(pts4, np.float32)
    assert p.ndim == 2 and p.shape[1] == 4
    n = p.shape[0]
    t_end = n if t_end is None else t_end
    e = np.zeros(max(t_end - t_begin, 1), np.float64)
    _check(lib().orc_triplet(n, _ptr(p), float(nu), t_begin, t_end, _ptr(e)))
    return e[: t_end - t_begin]


def triplet_abs(pts4: np.ndarray, nu: float = 1.0, t_begin: int = 0, t_end: int | None = None) -> np.ndarray:
    p = np.ascontiguousarray(pts4, np.float32)
    n = p.shape[0]
    t_end = n if t_end is None else t_end
    a = np.zeros(max(t_end - t_begin, 1), np.float64)
    _check(lib().orc_triplet_abs(n, _ptr(p), float(nu), t_begin, t_end, _ptr(a)))
    return a[: t_end - t_begin]


def triplet_total(pts4: np.ndarray, nu: float = 1.0) -> float:
    p = np.ascontiguousarray(pts4, np.float32)
    out = ctypes.c_double()
    _check(lib().orc_triplet_total(p.shape[0], _ptr(p), float(nu), ctypes.byref(out)))
    return out.value
