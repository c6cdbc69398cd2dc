"""Run tools/probes/f16acc.cu: TMEM layout of an F16 accumulator, and its precision:
is D(f16) = round_f16(exact K = 16 sum) (one rounding after a wide sum), or are partial
sums rounded to f16?  Prints the worst |D - exact| in units of the f16 ulp of D and
relative to sum |terms|, and sign mismatches."""
import ctypes, os
import numpy as np
import torch
L = ctypes.CDLL(os.path.join(os.getcwd(), "_ab", "libf16acc.so"))
st = torch.cuda.current_stream().cuda_stream


def run(A, B, dfmt):
    a = torch.from_numpy(A.astype(np.float16).view(np.int16).copy()).cuda()
    b = torch.from_numpy(B.astype(np.float16).view(np.int16).copy()).cuda()
    out = torch.zeros(128 * 256, dtype=torch.int32, device="cuda")
    rc = L.run_f16(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(out.data_ptr()), dfmt,
                   ctypes.c_void_p(st))
    torch.cuda.synchronize()
    assert rc == 0
    w = out.cpu().numpy().view(np.uint32).reshape(128, 256)
    if dfmt == 1:
        return w[:, :128].view(np.float32).astype(np.float64)
    return (w[:, :128] & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float64)


def packed_check():
    A = np.zeros((128, 16)); B = np.zeros((128, 16))
    A[:, 0] = 1; A[:, 1] = np.arange(128) / 256
    B[:, 0] = np.arange(128) / 128; B[:, 1] = 1
    a = torch.from_numpy(A.astype(np.float16).view(np.int16).copy()).cuda()
    b = torch.from_numpy(B.astype(np.float16).view(np.int16).copy()).cuda()
    out = torch.zeros(128 * 256, dtype=torch.int32, device="cuda")
    L.run_f16(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(out.data_ptr()), 0,
              ctypes.c_void_p(st))
    torch.cuda.synchronize()
    w = out.cpu().numpy().view(np.uint32).reshape(128, 256)
    D = (A @ B.T).astype(np.float16).view(np.uint16).astype(np.uint32)
    p = w[:, 128:144]
    ok = np.array_equal(p & 0xFFFF, D[:, 0:32:2]) and np.array_equal(p >> 16, D[:, 1:32:2])
    print("x16.pack::16b = columns (2c, 2c+1) in (lo, hi) halves:", ok, hex(int(p[5, 3])), hex(int(D[5, 6])), hex(int(D[5, 7])))


packed_check()


def f16(x):
    return np.asarray(x, np.float64).astype(np.float16).astype(np.float64)


rng = np.random.default_rng(1)
worst_ulp, worst_rel32, worst_rel16, signbad, n_eq_round = 0.0, 0.0, 0.0, 0, 0
tot = 0
for trial in range(24):
    sc = [0.5, 4.0, 0.01, 100.0][trial % 4]
    x = f16(rng.uniform(-sc, sc, (128, 3)))
    y = f16(x[rng.permutation(128)] + rng.normal(0, 1e-3 * sc, (128, 3)))
    y[:64] = x[:64]
    P = (x ** 2).sum(1); Q = (y ** 2).sum(1)
    def split(v):
        h = f16(v); m = f16(v - h); l = f16(v - h - m); return h, m, l
    Ph, Pm, Pl = split(P); Qh, Qm, Ql = split(Q)
    A = np.zeros((128, 16)); B = np.zeros((128, 16))
    A[:, :3] = x; A[:, 3], A[:, 4], A[:, 5] = Ph, Pm, Pl; A[:, 6:9] = 1
    B[:, :3] = f16(-2 * y); B[:, 3:6] = 1; B[:, 6], B[:, 7], B[:, 8] = Qh, Qm, Ql
    if trial % 3 == 2:                                    # random mixed-sign values too
        A = f16(rng.uniform(-2, 2, (128, 16))); B = f16(rng.uniform(-2, 2, (128, 16)))
    ex = A @ B.T
    ab = (np.abs(A)[:, None, :] * np.abs(B)[None, :, :]).sum(-1)
    d16 = run(A, B, 0)
    d32 = run(A, B, 1)
    fin = np.isfinite(d16)
    ulp = np.spacing(np.abs(f16(ex)).astype(np.float16)).astype(np.float64)
    err_ulp = np.abs(d16 - ex) / np.maximum(ulp, 2.0 ** -24)
    worst_ulp = max(worst_ulp, float(err_ulp[fin].max()))
    worst_rel16 = max(worst_rel16, float((np.abs(d16 - ex) / ab)[fin & (ab > 0)].max()))
    worst_rel32 = max(worst_rel32, float((np.abs(d32 - ex) / ab)[ab > 0].max()))
    signbad += int(((d16 < 0) != (ex < 0))[fin & (np.abs(ex) > 1e-6)].sum())
    n_eq_round += int((d16 == f16(d32))[fin].sum()); tot += int(fin.sum())
    bad = np.argwhere(fin & (d16 != f16(d32)))
    for (i, j) in bad[:4]:
        print(f"  trial {trial}: exact {ex[i, j]!r} d32 {d32[i, j]!r} d16 {d16[i, j]!r} round16(d32) {f16(d32[i, j])!r} sum|t| {ab[i, j]:.3g}")
    big = np.argwhere(fin & (np.abs(d16 - ex) > 1e-3 * ab))
    for (i, j) in big[:3]:
        print(f"  BIG trial {trial}: exact {ex[i, j]!r} d32 {d32[i, j]!r} d16 {d16[i, j]!r} sum|t| {ab[i, j]:.3g}")
print(f"F16 acc: worst |D - exact| = {worst_ulp:.2f} ulp(f16) ; relative to sum|terms| {worst_rel16:.3e}")
print(f"F32 acc: worst |D - exact| / sum|terms| = {worst_rel32:.3e}")
print(f"D16 == round_f16(D32) in {n_eq_round}/{tot}; sign mismatches (|exact| > 1e-6): {signbad}")
