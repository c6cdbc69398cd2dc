// collide_tc.cu -- TRI_LAMBDA_TC for tri_collide (rho = 256, 384 or 512): the collision
// filter gap of collide.cu evaluated on the 5th-generation tensor cores.
//
//   g_ij = A'_i + A'_j - 2 (x_i x_j + y_i y_j + z_i z_j + r_i r_j) = X_i . Y_j,
//   X_i = (x, y, z, r, A'_i, 1, 0, 0),  Y_j = (-2x, -2y, -2z, -2r, 1, A'_j, 0, 0)
//
// is a K = 8 contraction over the tile.  TF32 keeps 11 significant bits, so each
// operand is split into big + small TF32 parts and the tile is accumulated in
// TMEM from three kind::tf32 MMAs (X_big Y_big + X_big Y_small + X_small Y_big,
// 128 x 256 x 8 each): products of TF32 values are exact in fp32, the dropped
// small.small term is <= 2^-21 (M_i + M_j) and the fp32 accumulation adds a few
// ulps of sum |terms| <= 2 (M_i + M_j).  A' carries kappa u M with kappa u = 2^-15,
// so every pair the fixed-order predicate (reading Q9) counts still has g < 0;
// the epilogue ORs the sign bits of each row's 32-column groups and recounts a
// flagged group with the exact scalar predicate, so the count is exact.
//
// CTA = 128 threads (4 warps) per lambda tile; the tile is (rho/128)^2 blocks of
// 128 x 128, each one M = 128, N = 128 accumulator pass over 128 TMEM columns
// (larger tiles amortise the TMEM allocation and barrier set-up: rho = 256 2.83 ms,
// 512 2.41 ms (74 KB smem: 3 CTAs per SM), 384 2.24 ms (55 KB: 4 CTAs, as many as
// can hold their 128 TMEM columns at once)).
// Operands: K-major, no swizzle, canonical 8-row x 16-byte core matrices
// (LBO = 128 B between the two K halves, SBO = 256 B between 8-row groups).
// Diagonal tiles (strict j < i) are counted with the scalar predicate.
#include "tri_common.cuh"

namespace {

struct TcArgs {
    const float4 *sph;
    int64_t n;
    uint64_t omega_begin, omega_end;
    unsigned long long *count;
};

constexpr int kThreads = 128, kCols = 128;   // accumulator: 128 lanes x 128 fp32 columns
constexpr float kKappaU = 1.0f / 32768.0f;     // 2^-15

__device__ __forceinline__ float4 load_sph(const TcArgs &a, int64_t idx) {
    if (idx < a.n) return __ldg(a.sph + idx);
    const float nan = __int_as_float(0x7fffffff);
    return make_float4(nan, nan, nan, nan);
}

// The ABI's exact fixed-order predicate (reading Q9).
__device__ __forceinline__ uint32_t hit(const float4 p, const float4 q) {
    const float dx = __fsub_rn(p.x, q.x), dy = __fsub_rn(p.y, q.y), dz = __fsub_rn(p.z, q.z);
    const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
    const float s = __fadd_rn(p.w, q.w);
    return d2 < __fmul_rn(s, s) ? 1u : 0u;
}

__device__ __forceinline__ float a_prime(const float4 c) {
    const float q = fmaf(c.z, c.z, fmaf(c.y, c.y, c.x * c.x));
    const float w = c.w * c.w;
    return fmaf(-kKappaU, q + w, q - w);
}

__device__ __forceinline__ uint32_t tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

template <int kRho>
struct __align__(128) Smem {
    // operand rows: 32 B (K = 8 tf32) each, in the canonical core-matrix order
    uint32_t xb[kRho / 8][2][8][4], xs[kRho / 8][2][8][4];     // rows (A): big / small
    uint32_t yb[kRho / 8][2][8][4], ys[kRho / 8][2][8][4];     // cols (B): big / small
    float4 col[kRho];                                           // column spheres (exact recount)
    unsigned long long mbar;
    uint32_t taddr;
};

// store one operand row (8 values) split into big / small at row r of a [group][khalf][8][4] array
__device__ __forceinline__ void put_row(uint32_t (*big)[2][8][4], uint32_t (*sml)[2][8][4], int r,
                                        const float (&v)[8]) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t b = tf32(v[k]);
        big[r >> 3][k >> 2][r & 7][k & 3] = b;
        sml[r >> 3][k >> 2][r & 7][k & 3] = tf32(v[k] - __uint_as_float(b));
    }
}

__device__ __forceinline__ uint64_t smem_desc(const void *p) {
    const uint32_t addr = (uint32_t)__cvta_generic_to_shared(p);
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);            // start address
    d |= (uint64_t)(128 >> 4) << 16;                  // LBO: next K half
    d |= (uint64_t)(256 >> 4) << 32;                  // SBO: next 8-row group
    d |= (uint64_t)1 << 46;                           // version (Blackwell)
    return d;                                         // base offset 0, lbo mode 0, SWIZZLE_NONE
}

// kind::tf32, fp32 accumulator, K-major A and B, M = 128, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kCols >> 3) << 17) |
                            ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ bool mbar_wait(uint32_t mb, uint32_t parity) {
    for (int it = 0; it < (1 << 18); ++it) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(mb), "r"(parity)
            : "memory");
        if (done) return true;
    }
    return false;
}

template <int kRho>
__global__ void __launch_bounds__(kThreads) collide_tc_kernel(TcArgs a) {
    extern __shared__ __align__(128) unsigned char dsm[];
    Smem<kRho> &sm = *reinterpret_cast<Smem<kRho> *>(dsm);
    const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
    if (w >= a.omega_end) return;
    uint32_t bi, bj;
    tri::lambda_map(w, bi, bj);
    const int t = threadIdx.x, warp = t >> 5;
    const int64_t r0 = (int64_t)bi * kRho, c0 = (int64_t)bj * kRho;
    uint32_t cnt = 0;

    // columns: spheres for the recount, Y big / small operand rows
#pragma unroll
    for (int h = 0; h < kRho / kThreads; ++h) {
        const int j = t + kThreads * h;
        const float4 c = load_sph(a, c0 + j);
        sm.col[j] = c;
        const float v[8] = {-2.f * c.x, -2.f * c.y, -2.f * c.z, -2.f * c.w, 1.f, a_prime(c), 0.f, 0.f};
        put_row(sm.yb, sm.ys, j, v);
    }
    if (bi == bj) {                                      // diagonal tile: strict j < i, scalar exact
        __syncthreads();
#pragma unroll
        for (int h = 0; h < kRho / kThreads; ++h) {
            const int i = t + kThreads * h;
            const float4 p = load_sph(a, r0 + i);
#pragma unroll 4
            for (int j = 0; j < i; ++j) cnt += hit(p, sm.col[j]);
        }
    } else {
        // rows: X big / small operand rows (all 256; pass p uses rows 128 p ..)
        float4 prow[kRho / kThreads];
#pragma unroll
        for (int h = 0; h < kRho / kThreads; ++h) {
            const int i = t + kThreads * h;
            const float4 p = load_sph(a, r0 + i);
            prow[h] = p;
            const float v[8] = {p.x, p.y, p.z, p.w, a_prime(p), 1.f, 0.f, 0.f};
            put_row(sm.xb, sm.xs, i, v);
        }
        const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&sm.mbar);
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(&sm.taddr)),
                         "n"(kCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        if (t == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t tmem = sm.taddr;
        bool ok = true;
#pragma unroll 1
        for (int pass = 0; pass < (kRho / 128) * (kRho / 128); ++pass) {
            const int rh = pass / (kRho / 128), ch = pass % (kRho / 128);   // 128-row, 128-column block
            if (t == 0) {
                const int g0 = rh * 16, h0 = ch * 16;       // first 8-row groups of the A and B halves
                mma(tmem, smem_desc(&sm.xb[g0]), smem_desc(&sm.yb[h0]), 0u);
                mma(tmem, smem_desc(&sm.xb[g0]), smem_desc(&sm.ys[h0]), 1u);
                mma(tmem, smem_desc(&sm.xs[g0]), smem_desc(&sm.yb[h0]), 1u);
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    mb));
            }
            ok = mbar_wait(mb, (uint32_t)(pass & 1)) && ok;
            asm volatile("tcgen05.fence::after_thread_sync;");
            // epilogue: thread t = accumulator lane t = row 128 pass + t; 8 groups of 32 columns
            uint32_t flags = 0;
#pragma unroll
            for (int cg = 0; cg < kCols / 32; ++cg) {
                uint32_t v[32];
                const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(cg * 32);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                    "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                      "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
                      "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
                      "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(ta));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                uint32_t o = 0;                             // OR of 32 sign bits, 3-input LOP3s
#pragma unroll
                for (int e = 0; e < 32; e += 2)
                    asm("lop3.b32 %0, %1, %2, %3, 0xfe;" : "=r"(o) : "r"(o), "r"(v[e]), "r"(v[e + 1]));
                flags |= (o >> 31) << cg;
            }
            // rare: the exact predicate on this row's flagged 32-column groups
            const float4 p = prow[rh];
#pragma unroll 1
            while (flags) {
                const int cg = __ffs(flags) - 1;
                flags &= flags - 1;
#pragma unroll 4
                for (int j = 128 * ch + 32 * cg; j < 128 * ch + 32 * cg + 32; ++j) cnt += hit(p, sm.col[j]);
            }
            // every lane's loads are done before pass 1 overwrites the accumulator
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;");
        }
        if (warp == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
        // an MMA completion that never arrived (bounded wait): poison the count, never hang
        if (!ok && t == 0) atomicAdd(a.count, 1ull << 62);
    }
    // count: warp reduce, one atomic per warp (skipped if 0)
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((t & 31) == 0 && cnt) atomicAdd(a.count, (unsigned long long)cnt);
}

}  // namespace

namespace tri {

template <int kRho>
static void launch_rho(TcArgs a, uint64_t nb, cudaStream_t st) {
    const int smem = (int)sizeof(Smem<kRho>);
    cudaFuncSetAttribute(collide_tc_kernel<kRho>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    collide_tc_kernel<kRho><<<tile_grid(nb), kThreads, smem, st>>>(a);
}

tri_status launch_collide_tc(const tri_map_t &m, const float *sph, unsigned long long *count, cudaStream_t st) {
    if (m.rho != 256 && m.rho != 384 && m.rho != 512) return TRI_EINVAL;
    TcArgs a;
    a.sph = (const float4 *)sph;
    a.n = m.n;
    a.omega_begin = m.omega_begin;
    a.omega_end = m.omega_end;
    a.count = count;
    if (cudaMemsetAsync(count, 0, sizeof(unsigned long long), st) != cudaSuccess) return TRI_ECUDA;
    const uint64_t nb = a.omega_end - a.omega_begin;
    if (!nb) return TRI_OK;
    if (m.rho == 512) launch_rho<512>(a, nb, st);
    else if (m.rho == 384) launch_rho<384>(a, nb, st);
    else launch_rho<256>(a, nb, st);
    note_launches(1);
    return cuda_status();
}

}  // namespace tri
