// collide_tc.cu -- TRI_LAMBDA_TC / TRI_BB_TC for tri_collide (rho = 256, 384 or 512): the
// collision filter of reading Q9 evaluated on the 5th-generation tensor cores.
//
// The count is the fixed-order fp32 predicate d2 < s*s over j < i (reading
// Q9).  The tensor cores only FILTER: a pair the predicate counts always gets a negative
// filter value, and every (row, 32-column group) with a negative value is re-examined
// with the exact predicate, so the count is exact.
//
// Filter (one kind::tf32 MMA per 128 x 128 block, K = 8, every operand exact in TF32):
//   q_i  = tf32(p_i - c), c = (1/2, 1/2, 1/2)           quantised, centred position
//   e_i  = |p_i - (q_i + c)|                            its exact Euclidean error (fp64)
//   R_i  = tf32_up(r_i (1 + 8u) + e_i)                  inflated radius, u = 2^-24
//   A_i  = |q_i|^2 - R_i^2 - kappa u M_i,  M_i = |q_i|^2 + R_i^2   (fp64), split into
//          A_i = Ab_i + As_i + res_i with Ab, As TF32 and |res_i| <= 2^-21 M_i
//   X_i  = ( qx,  qy,  qz,  R, Ab, As, 1, 1)            row operand (A, K-major)
//   Y_j  = S (-2qx,-2qy,-2qz,-2R, 1,  1, Ab, As)        column operand (B, K-major), S = 2^20
//   g_ij = X_i . Y_j = S (|q_i - q_j|^2 - (R_i + R_j)^2 - kappa u (M_i + M_j) - res_i - res_j)
// (S is a power of two: exact, and it changes no sign.)
// Why it is conservative: the fp32 predicate counts only if the real distance satisfies
// d < (1 + 4.1u)(r_i + r_j) (three roundings in d2, two in s*s); then |q_i - q_j| <=
// d + e_i + e_j < R_i + R_j, so the exact value of X_i . Y_j is < -kappa u (M_i + M_j) +
// 2^-21 (M_i + M_j).  Products of TF32 values are exact in fp32; the tensor core's fp32
// sum of the 8 products is within 2^-20 sum_k |X_ik Y_jk| <= 2^-20 * 2.01 (M_i + M_j) of
// the exact sum (the accumulation bound, measured on B200 by tri_tc_tf32_probe and
// tests/test_gpu_parity.py::test_tc_tf32_accumulation_bound on adversarial cancelling
// operands).  With kappa u = 2^-16 the computed g_ij is therefore < 0.
//
// Layout: tri_collide's caller-owned workspace holds X and Y for m * rho rows (pad rows
// past n make every g positive) as canonical K-major no-swizzle core matrices: 8-row
// group g at byte 256 g, K half h at +128 h, row r at +16 r -- so a tile's operands are
// ONE contiguous rho x 32-byte run each, staged into shared memory by two 1-D bulk
// copies (cp.async.bulk, the TMA engine) completing on an mbarrier.
//
// CTA = 128 threads per tile (the paper's one block per lambda tile, Eq. 4, or the BB
// grid), 128 TMEM columns, 3 CTAs per SM.  Per 128 x 128 block one
// tcgen05.mma (issued by one thread) commits to an mbarrier; thread t = accumulator lane
// t = row t of the block loads all 128 columns into registers (4 x tcgen05.ld.32x32b.x32),
// the CTA hands the accumulator back (one barrier) and thread 0 issues the next block's
// MMA while every thread tests its values: 21 of each 32 by 3-input LOP3 ORs of the sign
// bits (ALU pipe), 11 by a saturating product P = sat(P g'), zero iff some g' <= 0 (FMA
// pipe; the MMA computes g' = 2^20 g so every pair that is not within 1e-6 of touching has
// g' >= 1 and leaves P = 1).  A flagged (row, 32-column group) recounts only its negative
// columns, from registers.  Diagonal tiles skip the blocks above the diagonal and recount
// j < i only.  Measured alternatives: persistent warp-specialised pipelines
// (one MMA warp, or self-issuing warpgroups), an issuer warp per tile with one or two
// accumulators, IMAD.HI sign counts -- all slower on B200.
#include "tri_common.cuh"

namespace {

constexpr int kThreads = 128, kCols = 128, kCtasPerSm = 3;
constexpr double kKappaU = 1.0 / 65536.0;               // 2^-16
constexpr float kPad = 1.0e30f;                         // pad-row operand: g = 1e30 > 0
constexpr float kScale = 1048576.0f;                    // S = 2^20: the column operand's scale

struct TcArgs {
    const float4 *sph;
    const uint32_t *ops;          // workspace: X rows [0, npad), then Y rows [0, npad)
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

__device__ __forceinline__ float tf32_rn(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// smallest TF32 value >= x (x >= 0, finite)
__device__ __forceinline__ float tf32_up(float x) {
    uint32_t b = __float_as_uint(x);
    if (b & 0x1fffu) b = (b | 0x1fffu) + 1u;
    return __uint_as_float(b);
}

// canonical K-major core-matrix slot of element k of row r
__device__ __forceinline__ int slot(int64_t r, int k) {
    return (int)(((r >> 3) * 64) + ((k >> 2) * 32) + ((r & 7) * 4) + (k & 3));
}

// ---------------------------------------------------------------- operand preparation
// One thread per row of [0, npad): the quantities of the header, in fp64 where an error
// bound is computed, written as TF32 bit patterns.  Thread 0 also zeroes the count.
__global__ void collide_tc_prep(const float4 *__restrict__ sph, int64_t n, int64_t npad, uint32_t *__restrict__ ops,
                                unsigned long long *count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) *count = 0ull;
    if (i >= npad) return;
    float x[8], y[8];
    if (i < n) {
        const float4 p = __ldg(sph + i);
        const float qx = tf32_rn(__fsub_rn(p.x, 0.5f)), qy = tf32_rn(__fsub_rn(p.y, 0.5f)),
                    qz = tf32_rn(__fsub_rn(p.z, 0.5f));
        // exact error of the quantised position: p, q and 1/2 are fp32, so every
        // difference and sum below is exact in fp64 (up to the final sqrt / square)
        const double ex = (double)p.x - ((double)qx + 0.5), ey = (double)p.y - ((double)qy + 0.5),
                     ez = (double)p.z - ((double)qz + 0.5);
        const double e = sqrt(ex * ex + ey * ey + ez * ez) * (1.0 + 0x1p-40) + 0x1p-60;
        const double r = fabs((double)p.w) * (1.0 + 0x1p-21) + e;     // (1 + 8u) r + e, rounded up below
        const float R = tf32_up(__double2float_ru(r));
        const double q2 = (double)qx * qx + (double)qy * qy + (double)qz * qz, R2 = (double)R * R;
        const double A = q2 - R2 - kKappaU * (q2 + R2);
        const float ab = tf32_rn((float)A);
        const float as = tf32_rn((float)(A - (double)ab));
        x[0] = qx; x[1] = qy; x[2] = qz; x[3] = R; x[4] = ab; x[5] = as; x[6] = 1.f; x[7] = 1.f;
        y[0] = -2.f * qx; y[1] = -2.f * qy; y[2] = -2.f * qz; y[3] = -2.f * R; y[4] = 1.f; y[5] = 1.f;
        y[6] = ab; y[7] = as;
#pragma unroll
        for (int k = 0; k < 8; ++k) y[k] *= kScale;
        if (A != A) {                                  // NaN: the predicate never counts it -> a pad row
#pragma unroll
            for (int k = 0; k < 8; ++k) { x[k] = 0.f; y[k] = 0.f; }
            x[4] = kPad;
            y[6] = kPad;
        } else if (!(fabs(A) < 1e30)) {                // huge: flagged against every real row / column
#pragma unroll
            for (int k = 0; k < 8; ++k) { x[k] = 0.f; y[k] = 0.f; }
            x[4] = -kPad;
            y[4] = kScale;
            y[6] = -kPad;
        }
    } else {                                           // pad row / column: g = 1e30 against real ones
#pragma unroll
        for (int k = 0; k < 8; ++k) { x[k] = 0.f; y[k] = 0.f; }
        x[4] = kPad;
        y[6] = kPad;
    }
    uint32_t *X = ops, *Y = ops + npad * 8;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        X[slot(i, k)] = __float_as_uint(x[k]);
        Y[slot(i, k)] = __float_as_uint(y[k]);
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

// kind::tf32, fp32 accumulator, K-major A and B, M = 128, N = kCols
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kCols >> 3) << 17) |
                            ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;\n\t}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(0), "r"(kIdesc));
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

__device__ __forceinline__ uint32_t or3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t o;
    asm("lop3.b32 %0, %1, %2, %3, 0xfe;" : "=r"(o) : "r"(a), "r"(b), "r"(c));
    return o;
}

__device__ __forceinline__ float mul_sat(float p, uint32_t g) {
    float r;
    asm("mul.rn.sat.f32 %0, %1, %2;" : "=f"(r) : "f"(p), "f"(__uint_as_float(g)));
    return r;
}

// The sign test of one 32-column group.  Values [0, 32 - kFmul): OR of their bit patterns
// by 3-input LOP3s (ALU pipe; bit 31 of `o` set iff one is negative).  Values
// [32 - kFmul, 32): P = sat(... sat(sat(1 g'_a) g'_b) ...) by saturating FMULs (FMA pipe):
// P stays in [0, 1] and is 0 iff some g' <= 0 (or P underflowed on values g' in (0, 1):
// only a false flag).  The group is flagged iff o < 0 or P == 0.
template <int kFmul>
struct Signs {
    uint32_t o;
    float p;
    __device__ __forceinline__ explicit Signs(const uint32_t (&v)[32]) {
        constexpr int kAlu = 32 - kFmul;
        static_assert(kAlu >= 3 && (kAlu - 3) % 2 == 0 && kFmul >= 1, "ALU share: 3 + 2k values");
        o = or3(v[0], v[1], v[2]);
#pragma unroll
        for (int e = 3; e < kAlu; e += 2) o = or3(o, v[e], v[e + 1]);
        float p0 = mul_sat(1.0f, v[kAlu]), p1 = 1.0f;
#pragma unroll
        for (int e = kAlu + 1; e < 32; ++e) {
            if ((e - kAlu) & 1) p1 = mul_sat(p1, v[e]);
            else p0 = mul_sat(p0, v[e]);
        }
        p = p0 * p1;
    }
    __device__ __forceinline__ bool flagged() const { return (int32_t)o < 0 || p == 0.0f; }
};

// bit e set iff value e of the group is negative (only for flagged groups: rare)
__device__ __forceinline__ uint32_t neg_mask(const uint32_t (&v)[32]) {
    uint32_t msk = 0;
#pragma unroll
    for (int e = 0; e < 32; ++e) msk |= (v[e] >> 31) << e;
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

template <int R>
__device__ __forceinline__ void block_of(bool diag, int idx, int &rh, int &ch) {
    if (diag) {                                        // triangular block index -> (rh, ch), ch <= rh
        rh = 0;
#pragma unroll
        for (int r = 1; r < R; ++r) rh += idx >= r * (r + 1) / 2;
        ch = idx - rh * (rh + 1) / 2;
    } else {
        rh = idx / R;
        ch = idx - rh * R;
    }
}

template <int kRho, bool kBB, int kFmul>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) collide_tc_kernel(TcArgs a) {
    constexpr int R = kRho / 128;
    constexpr uint32_t kOpBytes = kRho * 32;
    extern __shared__ __align__(1024) unsigned char dsm[];
    __shared__ __align__(8) unsigned long long mbar[2];     // [0] operands landed, [1] MMA done
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
    const uint32_t xs = (uint32_t)__cvta_generic_to_shared(dsm), ys = xs + kOpBytes;
    const uint32_t mb_ld = (uint32_t)__cvta_generic_to_shared(&mbar[0]);
    const uint32_t mb_mma = (uint32_t)__cvta_generic_to_shared(&mbar[1]);
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb_ld));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb_mma));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // the tile's operand rows: two contiguous runs of the workspace -> shared memory
        const uint32_t *gx = a.ops + (int64_t)bi * kRho * 8, *gy = a.ops + (a.npad + (int64_t)bj * kRho) * 8;
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
                     "n"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = taddr;
    const uint32_t lanes = tmem + ((uint32_t)(warp * 32) << 16);
    const bool diag = bi == bj;
    const int nblk = diag ? R * (R + 1) / 2 : R * R;
    auto issue = [&](int idx) {
        int rh, ch;
        block_of<R>(diag, idx, rh, ch);
        asm volatile("tcgen05.fence::after_thread_sync;");
        mma(tmem, smem_desc(xs + rh * 4096), smem_desc(ys + ch * 4096));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb_mma)
                     : "memory");
    };
    if (t == 0) {
        mbar_wait(mb_ld, 0, a.count);
        issue(0);
    }
    uint32_t cnt = 0;
#pragma unroll 1
    for (int idx = 0; idx < nblk; ++idx) {
        mbar_wait(mb_mma, (uint32_t)idx & 1u, a.count);
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint32_t v[4][32];
#pragma unroll
        for (int cg = 0; cg < 4; ++cg) ldtm32(lanes + (uint32_t)(cg * 32), v[cg]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // the accumulator is in registers: hand it back, the next MMA runs during the tests
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if (t == 0 && idx + 1 < nblk) issue(idx + 1);
        const Signs<kFmul> s0(v[0]), s1(v[1]), s2(v[2]), s3(v[3]);
        if ((int32_t)(or3(s0.o, s1.o, s2.o) | s3.o) < 0 || s0.p * s1.p * (s2.p * s3.p) == 0.0f) {   // rare
            int rh, ch;
            block_of<R>(diag, idx, rh, ch);
            const int64_t i = (int64_t)bi * kRho + rh * 128 + t;
            const int64_t j0 = (int64_t)bj * kRho + ch * 128;
            const int jlim = (diag && ch == rh) ? t : 128;   // strict j < i inside a diagonal block
            if (s0.flagged()) cnt += recount(a.sph, a.n, neg_mask(v[0]), i, j0, jlim);
            if (s1.flagged()) cnt += recount(a.sph, a.n, neg_mask(v[1]), i, j0 + 32, jlim - 32);
            if (s2.flagged()) cnt += recount(a.sph, a.n, neg_mask(v[2]), i, j0 + 64, jlim - 64);
            if (s3.flagged()) cnt += recount(a.sph, a.n, neg_mask(v[3]), i, j0 + 96, jlim - 96);
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((t & 31) == 0 && cnt) atomicAdd(a.count, (unsigned long long)cnt);
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

}  // namespace

namespace tri {

#ifndef TRI_TC_FMUL
#define TRI_TC_FMUL 1
#endif
constexpr int kFmul = TRI_TC_FMUL;   // values of each 32 tested on the FMA pipe (A/B'd on B200)

size_t collide_tc_ws_bytes(const tri_map_t &m) { return (size_t)m.m * (size_t)m.rho * 64u; }

template <int kRho, bool kBB>
static void launch_rho(const tri_map_t &m, TcArgs a, cudaStream_t st) {
    // pad the dynamic smem so at most kCtasPerSm CTAs share an SM (their TMEM columns fit)
    const int pad = 228 * 1024 / (kCtasPerSm + 1) + 1024;
    const int smem = 2 * kRho * 32 > pad ? 2 * kRho * 32 : pad;
    auto k = collide_tc_kernel<kRho, kBB, kFmul>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (kBB) k<<<dim3((unsigned)m.m, (unsigned)m.m), kThreads, smem, st>>>(a);
    else k<<<tile_grid(a.omega_end - a.omega_begin), kThreads, smem, st>>>(a);
}

tri_status launch_collide_tc(const tri_map_t &m, int strategy, const float *sph, unsigned long long *count,
                             void *ws, cudaStream_t st) {
    if (m.rho % 128 || m.rho < 256 || m.rho > 1024) return TRI_EINVAL;
    if (strategy == TRI_BB_TC && m.m > 65535) return TRI_EINVAL;
    TcArgs a;
    a.sph = (const float4 *)sph;
    a.ops = (const uint32_t *)ws;
    a.n = m.n;
    a.npad = m.m * (int64_t)m.rho;
    a.omega_begin = m.omega_begin;
    a.omega_end = m.omega_end;
    a.count = count;
    collide_tc_prep<<<(unsigned)((a.npad + 255) / 256), 256, 0, st>>>(a.sph, a.n, a.npad, (uint32_t *)ws, count);
    note_launches(1);
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

}  // namespace tri
