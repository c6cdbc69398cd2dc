// collide_tc.cu -- TRI_LAMBDA_TC / TRI_BB_TC for tri_collide (rho = 128 k, k = 2..8): the
// collision filter of reading Q9 evaluated on the 5th-generation tensor cores.
//
// The count is the fixed-order fp32 predicate d2 < s*s over j < i (reading
// Q9).  The tensor cores only FILTER: a pair the predicate counts always gets a negative
// filter value, and every (row, 32-column group) with a negative value is re-examined
// with the exact predicate, so the count is exact.
//
// Filter: one tcgen05.mma.kind::f16 per 128 x 128 block (fp16 operands, K = 16, of which
// 8 are used) into an F16 accumulator.  Every operand is an exact fp16 value:
//   2^-s        a power of two with |p - c| <= 1/2 and r <= 1/2 for every sphere after
//               scaling (collide_tc_bounds; c = (1/2, 1/2, 1/2); s = 0 on the unit cube)
//   q_i  = fp16((p_i - c) 2^-s)                       quantised, centred position
//   e_i  = |(p_i - c) 2^-s - q_i|                      its Euclidean error (fp64, + slack)
//   R_i  = fp16_up(r_i 2^-s (1 + 8u) + e_i)            inflated radius, u = 2^-24
//   A_i  = |q_i|^2 - R_i^2 - kappa_u M_i - kappa_a,    M_i = |q_i|^2 + R_i^2 (fp64),
//          = A1 + 2^-11 A2 + res, A1, A2 fp16, |res| <= 2^-24 |A| + 2^-36
//   X_i  = ( q,    R,    A1,  A2,      1,     2^-11, 0 ... 0)      (A operand, K-major)
//   Y_j  = S (-2q, -2R,  1,   2^-11,   A1_j,  A2_j,  0 ... 0)      (B operand), S = 2^15
//   g_ij = X_i . Y_j = S (|q_i - q_j|^2 - (R_i + R_j)^2 - kappa (..)_i - kappa (..)_j - res)
// Why it is conservative: the fp32 predicate counts only if the real distance d <
// (1 + 4.1u)(r_i + r_j) (three roundings in d2, two in s*s); then |q_i - q_j| <= d 2^-s +
// e_i + e_j < R_i + R_j, so the exact X_i . Y_j < -S (kappa_u (M_i + M_j) + 2 kappa_a -
// |res_i| - |res_j|) < -S kappa_u (M_i + M_j) / 2 - S kappa_a.  fp16 x fp16 products are
// exact; the tensor core sums them in (at least) fp32 precision -- within 2^-20 sum |terms|
// <= 2^-20 2.01 S (M_i + M_j) of the exact sum -- and rounds ONCE to the F16 accumulator
// (round to nearest, overflow to +-inf): both properties measured on B200
// (tests/test_gpu_tc.py::test_tc_tf32_accumulation_bound, test_tc_f16_accumulator_rounding,
// tools/probes/f16acc.cu).  With kappa_u = 2^-16 and kappa_a = 2^-24 the wide sum is below
// -S kappa_a = -2^-9, a normal fp16 value, so the F16 result keeps its sign bit.
// Pad rows past n and NaN spheres get operands that make every value positive; a sphere
// outside the scaled range (|q| > 1/2, R > 1/2: only non-finite or extreme inputs) is
// flagged against every row and column and decided by the exact predicate.
//
// Layout: tri_collide's caller-owned workspace = a 256-byte header (the bound) + X and Y
// for m * rho rows as canonical K-major no-swizzle core matrices (8-row group g at byte
// 256 g, K half h at +128 h, row r at +16 r: 32 bytes per row), so a tile's operands are
// ONE contiguous rho x 32-byte run each, staged into shared memory by two 1-D bulk copies
// (cp.async.bulk, the TMA engine) completing on an mbarrier.
//
// CTA = 256 sign-test threads + one issuer warp per tile (the paper's one block per lambda
// tile, Eq. 4, or the BB grid), 128 TMEM columns.  Per 128 x 128 block one MMA
// (issued by the issuer warp's lane 0) commits to an mbarrier; test threads t and t + 128 =
// accumulator lane t & 127 = row t & 127 of the block load one half of its 128 columns each
// (2 x tcgen05.ld.32x32b.x16.pack::16b: two F16 values per register, 32 registers), the CTA
// hands the accumulator back (one barrier) and the issuer issues the next block's MMA while
// every test thread ORs its 32 registers (16 three-input LOP3s: a quarter of an ALU op per
// pair) and tests bits 15 and 31.  A flagged (row, 32-column)
// group recounts only its negative columns with the exact predicate.  Diagonal tiles skip
// the blocks above the diagonal and recount j < i only.  (Round 2 history in DESIGN.md:
// the single-pass TF32 filter with F32 accumulators this replaces, persistent
// warp-specialised pipelines, issuer warps -- all measured slower.)
#include <cuda_fp16.h>
#include "tri_common.cuh"

namespace {

constexpr int kThreads = 128, kCols = 128;            // probes: one thread per accumulator lane
#ifndef TRI_TC_ISSUER
#define TRI_TC_ISSUER 1
#endif
// TRI_TC_ISSUER: one extra warp only issues the MMAs.  tcgen05.mma blocks the issuing thread
// until the tensor pipe accepts it (~250 clk behind the co-resident CTAs' MMAs, measured by
// clock64 tracing); in a sign-testing warp that delay lands on the CTA's critical path.
constexpr int kIssuer = TRI_TC_ISSUER;
#ifndef TRI_TC_ACCS
#define TRI_TC_ACCS 1
#endif
// accumulators per CTA: 2 = MMA b + 1 runs while the threads drain block b (ping-pong)
constexpr int kAccs = TRI_TC_ACCS;
#ifndef TRI_TC_N
#define TRI_TC_N 128
#endif
// Tile geometry: blocks of 128 rows x N columns, one tcgen05.mma (M = 128, N, K = 16) and one
// commit each (N = TRI_TC_N when it divides the tile edge, else 128).  Sign-test threads: warp w
// reads TMEM lane quarter w % 4 and the 64-column group w / 4, so 2 N test threads; TMEM
// N x kAccs columns per CTA, at most 512 per SM, which caps the CTAs per SM.
template <int kRho> struct TcCfg {
    static constexpr int N = (kRho % TRI_TC_N == 0) ? TRI_TC_N : 128;
    static constexpr int R = kRho / 128, CB = kRho / N;           // row / column blocks per tile
    static constexpr int TEST = 2 * N, THREADS = TEST + 32 * kIssuer;
    static constexpr int CTAS = 512 / (N * kAccs) < 8 ? 512 / (N * kAccs) : 8;
    // kind::f16: F16 accumulator (D format 0), F16 A and B (formats 0), K-major, M = 128, N
    static constexpr uint32_t IDESC = ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    static constexpr int diag_blocks() {                          // blocks of a diagonal tile
        int s = 0;
        for (int r = 0; r < R; ++r) s += (r * 128 + 127) / N + 1;
        return s;
    }
};
constexpr int kColsPerThread = 64;
static_assert(TRI_TC_N == 64 || TRI_TC_N == 128 || TRI_TC_N == 256, "MMA N");
constexpr double kKappaU = 1.0 / 65536.0;               // 2^-16 (relative margin)
constexpr double kKappaA = 1.0 / 16777216.0;            // 2^-24 (absolute margin, scaled units)
constexpr float kS = 32768.0f;                          // S = 2^15: the column operand's scale
constexpr float kPad = 60000.0f;                        // pad / extreme operand (fp16 range)
constexpr int kHdrBytes = 256;                          // workspace header: the bound

struct TcArgs {
    const float4 *sph;
    const uint16_t *ops;          // X rows [0, npad), then Y rows [0, npad): 16 halves each
    int64_t n, npad;
    uint64_t omega_begin, omega_end;
    unsigned long long *count;
};

// The ABI's exact fixed-order predicate (reading Q9).
__device__ __forceinline__ uint32_t hit(const float4 p, const float4 q) {
    const float dx = __fsub_rn(p.x, q.x), dy = __fsub_rn(p.y, q.y), dz = __fsub_rn(p.z, q.z);
    const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
    const float s = __fadd_rn(p.w, q.w);
    return d2 < __fmul_rn(s, s) ? 1u : 0u;
}

// canonical K-major core-matrix slot (in halves) of element k (0..15) of row r
__device__ __forceinline__ int64_t slot16(int64_t r, int k) {
    return ((r >> 3) * 128) + ((k >> 3) * 64) + ((r & 7) * 8) + (k & 7);
}

// ---------------------------------------------------------------- operand preparation
// hdr[0] = max over spheres of max(|x - 1/2|, |y - 1/2|, |z - 1/2|, |r|) as float bits
// (non-negative floats order like their bit patterns; NaN is skipped).  Thread 0 also
// zeroes the count.  hdr[0] is zeroed by the launcher before this kernel.
__global__ void collide_tc_bounds(const float4 *__restrict__ sph, int64_t n, uint32_t *hdr,
                                  unsigned long long *count) {
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i0 == 0) *count = 0ull;
    float b = 0.f;
    for (int64_t i = i0; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 p = __ldg(sph + i);
        b = fmaxf(b, fmaxf(fmaxf(fabsf(p.x - 0.5f), fabsf(p.y - 0.5f)), fmaxf(fabsf(p.z - 0.5f), fabsf(p.w))));
    }
    b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, 16));
    b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, 8));
    b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, 4));
    b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, 2));
    b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, 1));
    if ((threadIdx.x & 31) == 0 && b > 0.f) atomicMax(hdr, __float_as_uint(b));
}

// One thread per row of [0, npad): the quantities of the header, in fp64 where an error
// bound is computed, written as fp16 bit patterns.
__global__ void collide_tc_prep(const float4 *__restrict__ sph, int64_t n, int64_t npad, const uint32_t *hdr,
                                uint16_t *__restrict__ ops) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npad) return;
    // the scale 2^-s: |p - c| 2^-s <= 1/2 and r 2^-s <= 1/2 (bound = m 2^e, m in [1/2, 1))
    const float bound = __uint_as_float(*hdr);
    int s = 0;
    if (bound > 0.5f && bound < 1e30f) {
        int e;
        frexpf(bound, &e);
        s = e + 1;
    }
    const double sc = ldexp(1.0, -s);
    float x[16], y[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) { x[k] = 0.f; y[k] = 0.f; }
    bool pad = i >= n, extreme = false;
    if (!pad) {
        const float4 p = __ldg(sph + i);
        const double px = ((double)p.x - 0.5) * sc, py = ((double)p.y - 0.5) * sc, pz = ((double)p.z - 0.5) * sc;
        const __half qx = __double2half(px), qy = __double2half(py), qz = __double2half(pz);
        const double fx = __half2float(qx), fy = __half2float(qy), fz = __half2float(qz);
        const double ex = px - fx, ey = py - fy, ez = pz - fz;
        // + slack for the (p - 1/2) sc rounding in fp64 (relative 2^-53) and the sqrt
        const double e = sqrt(ex * ex + ey * ey + ez * ez) * (1.0 + 0x1p-40) +
                         (fabs(px) + fabs(py) + fabs(pz)) * 0x1p-50 + 0x1p-60;
        const double rr = fabs((double)p.w) * sc * (1.0 + 0x1p-21) + e;
        const __half R = __float2half_ru(__double2float_ru(rr));
        const double fR = __half2float(R);
        const double q2 = fx * fx + fy * fy + fz * fz, R2 = fR * fR;
        const double A = q2 - R2 - kKappaU * (q2 + R2) - kKappaA;
        if (p.x != p.x || p.y != p.y || p.z != p.z || p.w != p.w) {
            pad = true;                                   // NaN: the predicate never counts it
        } else if (!(fabs(fx) <= 0.5 && fabs(fy) <= 0.5 && fabs(fz) <= 0.5 && fR <= 0.5)) {
            extreme = true;
        } else {
            const __half a1 = __double2half(A);
            const __half a2 = __double2half((A - (double)__half2float(a1)) * 2048.0);
            const float A1 = __half2float(a1), A2 = __half2float(a2);
            x[0] = (float)fx; x[1] = (float)fy; x[2] = (float)fz; x[3] = (float)fR;
            x[4] = A1; x[5] = A2; x[6] = 1.f; x[7] = 1.f / 2048.f;
            y[0] = -2.f * kS * (float)fx; y[1] = -2.f * kS * (float)fy; y[2] = -2.f * kS * (float)fz;
            y[3] = -2.f * kS * (float)fR; y[4] = kS; y[5] = kS / 2048.f; y[6] = kS * A1; y[7] = kS * A2;
        }
    }
    if (pad) {                                            // g = +60000 S against real rows / columns
        x[4] = kPad;
        y[6] = kPad;
    } else if (extreme) {                                 // g < 0 against every real row / column
        x[4] = -kPad;
        y[4] = 1.f;
        y[6] = -kPad;
    }
    uint16_t *X = ops, *Y = ops + npad * 16;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        X[slot16(i, k)] = __half_as_ushort(__float2half_rn(x[k]));   // every value is an exact fp16
        Y[slot16(i, k)] = __half_as_ushort(__float2half_rn(y[k]));
    }
}

// ---------------------------------------------------------------- tcgen05 / TMA helpers
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);            // start address
    d |= (uint64_t)(128 >> 4) << 16;                  // LBO: next K half
    d |= (uint64_t)(256 >> 4) << 32;                  // SBO: next 8-row group
    d |= (uint64_t)1 << 46;                           // version (Blackwell)
    return d;                                         // base offset 0, lbo mode 0, SWIZZLE_NONE
}

// kind::f16: F16 accumulator (D format 0), F16 A and B (formats 0), K-major, M = 128, N = kCols
constexpr uint32_t kIdescF16 = ((uint32_t)(kCols >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
// kind::tf32, F32 accumulator (the accumulation probe)
constexpr uint32_t kIdescTf32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kCols >> 3) << 17) |
                                ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void mma_f16(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc = kIdescF16) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n\t}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(0), "r"(idesc));
}

__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;\n\t}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(0), "r"(kIdescTf32));
}

// Wait for an mbarrier phase (the thread parks on the barrier until the phase completes or
// the suspend-time hint expires).  A completion that never arrives (a broken tensor-core
// or copy path) must not hang the GPU or leave a plausible count: after ~2 s the count
// gets its sticky invalid bit 63 (include/tri.h) and the kernel traps.
__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t parity, unsigned long long *count) {
    long long t0 = 0;
    for (int it = 0;; ++it) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.b32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(mb), "r"(parity), "r"(0x989680)
            : "memory");
        if (done) return;
        if (it == 8) t0 = clock64();
        if (it > 8 && (it & 15) == 0 && clock64() - t0 > 4000000000ll) {
            if (count) atomicOr(count, 1ull << 63);
            __trap();
        }
    }
}

__device__ __forceinline__ void ldtm32(uint32_t ta, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
          "=r"(v[30]), "=r"(v[31])
        : "r"(ta));
}

// 32 F16 accumulator columns into 16 registers: column 2c in the low half of v[c], 2c + 1 in the high
__device__ __forceinline__ void ldtm16p(uint32_t ta, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(ta));
}

__device__ __forceinline__ uint32_t or3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t o;
    asm("lop3.b32 %0, %1, %2, %3, 0xfe;" : "=r"(o) : "r"(a), "r"(b), "r"(c));
    return o;
}

// OR of 16 packed registers (32 F16 values): bit 15 / 31 set iff some even / odd column is negative
__device__ __forceinline__ uint32_t or16(const uint32_t (&v)[16]) {
    uint32_t o = or3(v[0], v[1], v[2]);
#pragma unroll
    for (int e = 3; e < 15; e += 2) o = or3(o, v[e], v[e + 1]);
    return o | v[15];
}

// bit e set iff column e of the 32-column group is negative (only for flagged groups: rare)
__device__ __forceinline__ uint32_t neg_mask16(const uint32_t (&v)[16]) {
    uint32_t msk = 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) msk |= (((v[c] >> 15) & 1u) << (2 * c)) | ((v[c] >> 31) << (2 * c + 1));
    return msk;
}

// the exact predicate on the negative columns of one flagged group, j0 + e for the set
// bits e of msk below jlim (rare: not inlined, keeps the hot loop small)
__device__ __noinline__ uint32_t recount(const float4 *sph, int64_t n, uint32_t msk, int64_t i, int64_t j0,
                                         int jlim) {
    if (jlim < 32) msk &= jlim <= 0 ? 0u : (1u << jlim) - 1u;
    if (!msk || i >= n) return 0;
    const float4 p = __ldg(sph + i);
    uint32_t cnt = 0;
    while (msk) {
        const int e = __ffs(msk) - 1;
        msk &= msk - 1;
        if (j0 + e < n) cnt += hit(p, __ldg(sph + j0 + e));
    }
    return cnt;
}

// block index -> (row block rh, column block ch); a diagonal tile has only the blocks that
// reach the lower triangle (ch N <= 128 rh + 127)
template <class C>
__device__ __forceinline__ void block_of(bool diag, int idx, int &rh, int &ch) {
    if (diag) {
        rh = 0;
        int base = 0;
        bool done = false;
#pragma unroll
        for (int r = 0; r < C::R; ++r) {
            const int c = (r * 128 + 127) / C::N + 1;
            if (!done && idx >= base + c) {
                base += c;
                rh = r + 1;
            } else {
                done = true;
            }
        }
        ch = idx - base;
    } else {
        rh = idx / C::CB;
        ch = idx - rh * C::CB;
    }
}

template <int kRho, bool kBB>
__global__ void __launch_bounds__(TcCfg<kRho>::THREADS, TcCfg<kRho>::CTAS) collide_tc_kernel(TcArgs a) {
    using C = TcCfg<kRho>;
    constexpr uint32_t kOpBytes = kRho * 32;
    extern __shared__ __align__(1024) unsigned char dsm[];
    __shared__ __align__(8) unsigned long long mbar[1 + kAccs];   // [0] operands landed, [1 + a] MMA into acc a done
    __shared__ uint32_t taddr;
    uint32_t bi, bj;
    if (kBB) {                                         // m x m grid: blocks above the diagonal exit
        bj = blockIdx.x;
        bi = blockIdx.y;
        if (bj > bi) return;
        const uint64_t w = tri::T2(bi) + bj;
        if (w < a.omega_begin || w >= a.omega_end) return;
    } else {
        const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (w >= a.omega_end) return;
        tri::lambda_map(w, bi, bj);
    }
    const int t = threadIdx.x, warp = t >> 5;
    constexpr int kIssueT = kIssuer ? C::TEST : 0;           // the thread that issues copies and MMAs
    const bool issuer_warp = kIssuer && t >= C::TEST;
    const uint32_t xs = (uint32_t)__cvta_generic_to_shared(dsm), ys = xs + kOpBytes;
    const uint32_t mb_ld = (uint32_t)__cvta_generic_to_shared(&mbar[0]);
    const uint32_t mb_mma = (uint32_t)__cvta_generic_to_shared(&mbar[1]);   // + 8 acc
    if (t == kIssueT) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb_ld));
#pragma unroll
        for (int q = 0; q < kAccs; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb_mma + 8 * q));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // the tile's operand rows: two contiguous runs of the workspace -> shared memory
        const uint16_t *gx = a.ops + (int64_t)bi * kRho * 16, *gy = a.ops + (a.npad + (int64_t)bj * kRho) * 16;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb_ld), "r"(2 * kOpBytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(xs),
            "l"(gx), "r"(kOpBytes), "r"(mb_ld)
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(ys),
            "l"(gy), "r"(kOpBytes), "r"(mb_ld)
            : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&taddr)),
                     "n"(C::N * kAccs));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = taddr;
    const int row = t & 127, colbase = (warp >> 2) * kColsPerThread;   // accumulator lane, first column
    const uint32_t lanes = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)colbase;
    const bool diag = bi == bj;
    const int nblk = diag ? C::diag_blocks() : C::R * C::CB;
    auto issue = [&](int idx) {
        int rh, ch;
        block_of<C>(diag, idx, rh, ch);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int acc = kAccs == 1 ? 0 : (idx & 1);
        mma_f16(tmem + (uint32_t)(acc * C::N), smem_desc(xs + rh * 4096), smem_desc(ys + ch * C::N * 32), C::IDESC);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         mb_mma + 8 * acc)
                     : "memory");
    };
    if (t == kIssueT) {
        mbar_wait(mb_ld, 0, a.count);
        issue(0);
        if (kAccs == 2 && nblk > 1) issue(1);
    }
    uint32_t cnt = 0;
    if (issuer_warp) {
        // the issuer warp: one hand-back barrier per block, then the next MMA
#pragma unroll 1
        for (int idx = 0; idx < nblk; ++idx) {
            __syncthreads();
            if (t == kIssueT && idx + kAccs < nblk) issue(idx + kAccs);
        }
    } else {
#pragma unroll 1
    for (int idx = 0; idx < nblk; ++idx) {
        const int acc = kAccs == 1 ? 0 : (idx & 1);
        mbar_wait(mb_mma + 8 * acc, (uint32_t)(kAccs == 1 ? idx : idx >> 1) & 1u, a.count);
        asm volatile("tcgen05.fence::after_thread_sync;");
        constexpr int NG = kColsPerThread / 32;            // 32-column groups per thread
        uint32_t v[NG][16];
#pragma unroll
        for (int cg = 0; cg < NG; ++cg) ldtm16p(lanes + (uint32_t)(acc * C::N + cg * 32), v[cg]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // the accumulator is in registers: hand it back, the next MMA runs during the tests
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if (!kIssuer && t == 0 && idx + kAccs < nblk) issue(idx + kAccs);
        uint32_t o[NG], any = 0;
#pragma unroll
        for (int cg = 0; cg < NG; ++cg) { o[cg] = or16(v[cg]); any |= o[cg]; }
        if (any & 0x80008000u) {                           // rare: some value of the row is negative
            int rh, ch;
            block_of<C>(diag, idx, rh, ch);
            const int64_t i = (int64_t)bi * kRho + rh * 128 + row;
            const int64_t j0 = (int64_t)bj * kRho + ch * C::N + colbase;
            // strict j < i inside a diagonal tile: tile column ch N + colbase + e < tile row 128 rh + row
            const int jlim = diag ? rh * 128 + row - (ch * C::N + colbase) : kColsPerThread;
#pragma unroll
            for (int cg = 0; cg < NG; ++cg)
                if (o[cg] & 0x80008000u) cnt += recount(a.sph, a.n, neg_mask16(v[cg]), i, j0 + 32 * cg, jlim - 32 * cg);
        }
    }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::N * kAccs));
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((t & 31) == 0 && cnt) atomicAdd(a.count, (unsigned long long)cnt);
}

// canonical K-major core-matrix slot of 32-bit element k (0..7) of row r (the TF32 probe)
__device__ __forceinline__ int slot(int64_t r, int k) {
    return (int)(((r >> 3) * 64) + ((k >> 2) * 32) + ((r & 7) * 4) + (k & 3));
}

// ---------------------------------------------------------------- accumulation probe
// D = X Y^T for one 128 x 128 x 8 block with caller-given TF32 operands (row-major
// 128 x 8 each): the raw tensor-core fp32 result, for the accumulation-bound test.
__global__ void __launch_bounds__(kThreads) tc_tf32_probe_kernel(const float *x, const float *y, float *d) {
    __shared__ __align__(1024) uint32_t sx[128 * 8], sy[128 * 8];
    __shared__ __align__(8) unsigned long long mbar;
    __shared__ uint32_t taddr;
    const int t = threadIdx.x, warp = t >> 5;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        sx[slot(t, k)] = __float_as_uint(x[t * 8 + k]);
        sy[slot(t, k)] = __float_as_uint(y[t * 8 + k]);
    }
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&taddr)),
                     "n"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = taddr;
    if (t == 0) {
        mma(tmem, smem_desc((uint32_t)__cvta_generic_to_shared(sx)), smem_desc((uint32_t)__cvta_generic_to_shared(sy)));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb)
                     : "memory");
    }
    mbar_wait(mb, 0, nullptr);
    asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
    for (int cg = 0; cg < kCols / 32; ++cg) {
        uint32_t v[32];
        ldtm32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(cg * 32), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int e = 0; e < 32; ++e) d[t * 128 + cg * 32 + e] = __uint_as_float(v[e]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
}

// D = X Y^T for one 128 x 128 x 16 block with caller-given fp16 operands (row-major
// 128 x 16 each) into an F16 accumulator, read back with the packed loads the filter
// uses: the accumulator-rounding test (d: 128 x 128 fp16 bit patterns).
__global__ void __launch_bounds__(kThreads) tc_f16_probe_kernel(const uint16_t *x, const uint16_t *y, uint16_t *d) {
    __shared__ __align__(1024) uint16_t sx[128 * 16], sy[128 * 16];
    __shared__ __align__(8) unsigned long long mbar;
    __shared__ uint32_t taddr;
    const int t = threadIdx.x, warp = t >> 5;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        sx[slot16(t, k)] = x[t * 16 + k];
        sy[slot16(t, k)] = y[t * 16 + k];
    }
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&taddr)),
                     "n"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = taddr;
    if (t == 0) {
        mma_f16(tmem, smem_desc((uint32_t)__cvta_generic_to_shared(sx)),
                smem_desc((uint32_t)__cvta_generic_to_shared(sy)));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb)
                     : "memory");
    }
    mbar_wait(mb, 0, nullptr);
    asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
    for (int cg = 0; cg < kCols / 32; ++cg) {
        uint32_t v[16];
        ldtm16p(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(cg * 32), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            d[t * 128 + cg * 32 + 2 * c] = (uint16_t)(v[c] & 0xffffu);
            d[t * 128 + cg * 32 + 2 * c + 1] = (uint16_t)(v[c] >> 16);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
}

}  // namespace

namespace tri {

size_t collide_tc_ws_bytes(const tri_map_t &m) { return (size_t)kHdrBytes + (size_t)m.m * (size_t)m.rho * 64u; }

template <int kRho, bool kBB>
static void launch_rho(const tri_map_t &m, TcArgs a, cudaStream_t st) {
    using C = TcCfg<kRho>;
    // pad the dynamic smem so at most C::CTAS CTAs share an SM (their TMEM columns fit)
    const int pad = 228 * 1024 / (C::CTAS + 1) + 1024;
    const int smem = 2 * kRho * 32 > pad ? 2 * kRho * 32 : pad;
    auto k = collide_tc_kernel<kRho, kBB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (kBB) k<<<dim3((unsigned)m.m, (unsigned)m.m), C::THREADS, smem, st>>>(a);
    else k<<<tile_grid(a.omega_end - a.omega_begin), C::THREADS, smem, st>>>(a);
}

tri_status launch_collide_tc(const tri_map_t &m, int strategy, const float *sph, unsigned long long *count,
                             void *ws, cudaStream_t st) {
    if (m.rho % 128 || m.rho < 256 || m.rho > 1024) return TRI_EINVAL;
    if (strategy == TRI_BB_TC && m.m > 65535) return TRI_EINVAL;
    TcArgs a;
    a.sph = (const float4 *)sph;
    a.ops = (const uint16_t *)((const uint8_t *)ws + kHdrBytes);
    a.n = m.n;
    a.npad = m.m * (int64_t)m.rho;
    a.omega_begin = m.omega_begin;
    a.omega_end = m.omega_end;
    a.count = count;
    uint32_t *hdr = (uint32_t *)ws;
    if (cudaMemsetAsync(hdr, 0, sizeof(uint32_t), st) != cudaSuccess) return TRI_ECUDA;
    const int gb = (int)((a.n + 255) / 256 < 2 * (int64_t)sm_count() ? (a.n + 255) / 256 : 2 * sm_count());
    collide_tc_bounds<<<gb > 0 ? gb : 1, 256, 0, st>>>(a.sph, a.n, hdr, count);
    collide_tc_prep<<<(unsigned)((a.npad + 255) / 256), 256, 0, st>>>(a.sph, a.n, a.npad, hdr,
                                                                      (uint16_t *)((uint8_t *)ws + kHdrBytes));
    note_launches(2);
    if (a.omega_end > a.omega_begin) {
        const bool bb = strategy == TRI_BB_TC;
        if (m.rho == 1024) bb ? launch_rho<1024, true>(m, a, st) : launch_rho<1024, false>(m, a, st);
        else if (m.rho == 896) bb ? launch_rho<896, true>(m, a, st) : launch_rho<896, false>(m, a, st);
        else if (m.rho == 768) bb ? launch_rho<768, true>(m, a, st) : launch_rho<768, false>(m, a, st);
        else if (m.rho == 640) bb ? launch_rho<640, true>(m, a, st) : launch_rho<640, false>(m, a, st);
        else if (m.rho == 512) bb ? launch_rho<512, true>(m, a, st) : launch_rho<512, false>(m, a, st);
        else if (m.rho == 384) bb ? launch_rho<384, true>(m, a, st) : launch_rho<384, false>(m, a, st);
        else bb ? launch_rho<256, true>(m, a, st) : launch_rho<256, false>(m, a, st);
        note_launches(1);
    }
    return cuda_status();
}

tri_status launch_tc_tf32_probe(const float *x, const float *y, float *d, cudaStream_t st) {
    tc_tf32_probe_kernel<<<1, kThreads, 0, st>>>(x, y, d);
    note_launches(1);
    return cuda_status();
}

tri_status launch_tc_f16_probe(const void *x, const void *y, void *d, cudaStream_t st) {
    tc_f16_probe_kernel<<<1, kThreads, 0, st>>>((const uint16_t *)x, (const uint16_t *)y, (uint16_t *)d);
    note_launches(1);
    return cuda_status();
}

}  // namespace tri
