"""Run tools/probes/f16acc.cu: TMEM layout of an F16 accumulator, and its precision."""
import ctypes, os
import numpy as np
import torch
L = ctypes.CDLL(os.path.join(os.getcwd(), "_ab", "libf16acc.so"))
st = torch.cuda.current_stream().cuda_stream


def run(A, B, dfmt):
    a = torch.from_numpy(A.astype(np.float16).view(np.uint16).astype(np.int16)).cuda()
    b = torch.from_numpy(B.astype(np.float16).view(np.uint16).astype(np.int16)).cuda()
    out = torch.zeros(128 * 256, dtype=torch.int32, device="cuda")
    rc = L.run_f16(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(out.data_ptr()), dfmt,
                   ctypes.c_void_p(st))
    torch.cuda.synchronize()
    assert rc == 0
    return out.cpu().numpy().view(np.uint32).reshape(128, 256)


# 1. layout
A = np.zeros((128, 16)); B = np.zeros((128, 16))
A[:, 0] = 1; A[:, 1] = np.arange(128) / 256
B[:, 0] = np.arange(128) / 128; B[:, 1] = 1
D = A @ B.T
for dfmt in (1, 0):
    w = run(A, B, dfmt)
    used = [c for c in range(256) if (w[:, c] != 0xDEADBEEF).any()]
    print(f"dfmt={dfmt}: columns written: {used[0]}..{used[-1]} ({len(used)} cols)")
    if dfmt == 1:
        f = w[:, :128].view(np.float32)
        print("  f32 matches D:", np.array_equal(f, D.astype(np.float32)))
    else:
        lo = (w[:, :64] & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float64)
        hi = (w[:, :64] >> 16).astype(np.uint16).view(np.float16).astype(np.float64)
        print("  packed (lo=col 2c, hi=col 2c+1):", np.array_equal(lo, D[:, 0::2]) and np.array_equal(hi, D[:, 1::2]))
        lo2 = (w[:, :128] & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float64)
        print("  unpacked (lo half of col c):", np.array_equal(lo2, D), " hi halves:", hex(int(w[0, 0] >> 16)))
        print("  row0 words:", [hex(x) for x in w[0, :4]], "D row0:", D[0, :4])

# 2. precision of the F16 output on cancelling operands (fp16 exact inputs)
rng = np.random.default_rng(1)
worst_rel, worst_abs, signbad = 0.0, 0.0, 0
for trial in range(20):
    sc = [0.5, 4.0, 0.01, 100.0][trial % 4]
    x = rng.uniform(-sc, sc, (128, 3)).astype(np.float16).astype(np.float64)
    y = (x[rng.permutation(128)] + rng.normal(0, 1e-3 * sc, (128, 3))).astype(np.float16).astype(np.float64)
    y[:64] = x[:64]
    P = (x ** 2).sum(1); Q = (y ** 2).sum(1)
    def split(v):
        h = v.astype(np.float16).astype(np.float64); m = (v - h).astype(np.float16).astype(np.float64)
        l = (v - h - m).astype(np.float16).astype(np.float64); return h, m, l
    Ph, Pm, Pl = split(P); Qh, Qm, Ql = split(Q)
    A = np.zeros((128, 16)); B = np.zeros((128, 16))
    A[:, :3] = x; A[:, 3], A[:, 4], A[:, 5] = Ph, Pm, Pl; A[:, 6:9] = 1
    B[:, :3] = (-2 * y).astype(np.float16); B[:, 3:6] = 1; B[:, 6], B[:, 7], B[:, 8] = Qh, Qm, Ql
    A = A.astype(np.float16).astype(np.float64); B = B.astype(np.float16).astype(np.float64)
    ex = A @ B.T
    ab = np.abs(A)[:, None, :] * np.abs(B)[None, :, :]
    ab = ab.sum(-1)
    w = run(A, B, 0)
    lo = (w[:, :64] & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float64)
    hi = (w[:, :64] >> 16).astype(np.uint16).view(np.float16).astype(np.float64)
    got = np.empty((128, 128)); got[:, 0::2] = lo; got[:, 1::2] = hi
    sgn_got = np.signbit(np.concatenate([(w[:, :64] & 0x8000) != 0, (w[:, :64] & 0x80000000) != 0], 1))
    nz = ex != 0
    rel = np.abs(got - ex) / np.maximum(np.abs(ex), 6.1e-5)
    worst_rel = max(worst_rel, float(rel[nz].max()))
    worst_abs = max(worst_abs, float((np.abs(got - ex) / ab).max()))
    signbad += int(((got < 0) != (ex < 0))[np.abs(ex) > 1e-7].sum())
    w32 = run(A, B, 1)[:, :128].view(np.float32).astype(np.float64)
    if trial == 0:
        print("f32 acc: max |err|/sum|terms| =", float((np.abs(w32 - ex) / ab).max()))
print(f"F16 acc: worst |err|/max(|exact|, 6.1e-5) = {worst_rel:.3e} (single final rounding: <= 2^-11 = {2**-11:.3e}); "
      f"worst |err|/sum|terms| = {worst_abs:.3e}; sign mismatches (|exact| > 1e-7): {signbad}")
