// collide.cu -- all-pairs sphere collision count over the strict lower
// triangle ("collision detection of N spheres with random
// radius inside a unit box ... using a shared memory approach").
//
// Tile = rho x rho sphere pairs, coordinate from lambda(omega) or the BB grid.
// The rho column spheres of the tile are staged in shared memory as five
// arrays (-2x, -2y, -2z, -2r, A'): an aligned LDS.128 of one array is two packed
// f32x2 operands (columns c, c+1 and c+2, c+3), 20 B per sphere.  Each of the
// rho/K threads holds K row spheres (K = 8 at rho >= 256, else 4), each
// duplicated into both halves of an f32x2, and tests them against every column
// pair with the sm_100 packed FFMA2 / FADD2 instructions.  The count is the
// ABI's fixed scalar predicate (reading Q9):
//   dx = xi - xj, dy, dz;  d2 = fma(dz,dz, fma(dy,dy, dx*dx));  s = ri + rj;  d2 < s*s
// but hits are rare (~6e-6 of the pairs at the benchmark), so the hot loop only
// FILTERS: per 32-column block each thread keeps a bit per column whose gap
// (below) is negative for one of its rows, and only flagged columns are
// recounted with the exact predicate.  The gap is d2 - s^2 expanded around the
// origin as a 4-D dot product,
//   d2 - s^2 = A_i + A_j - 2 (x_i x_j + y_i y_j + z_i z_j + r_i r_j),
//   A = |x|^2 - r^2,
// evaluated as g = A'_i + fma(x_i, -2x_j, fma(y_i, -2y_j, fma(z_i, -2z_j,
// fma(r_i, -2r_j, A'_j)))) -- 5 FP32 ops per pair instead of the predicate's 9
// -- with A' = A - kappa u M, M = |x|^2 + r^2, u = 2^-24, kappa = 64.  The
// filter's rounding error is <= ~15 u (M_i + M_j) and a pair the fixed-order
// predicate counts has d2* - s*^2 <= ~10 u (M_i + M_j) in exact arithmetic
// (first order), so every counted pair has
// g < (25 - kappa) u (M_i + M_j) < 0: no hit is ever missed, and the count is
// exactly the predicate's.  The per-sphere A' is computed while staging the
// tile.  NaN (out-of-range spheres) never flags (min ignores NaN).  Diagonal
// tiles use the scalar predicate with the strict filter col < row.  Counts are
// reduced per warp and CTA; one 64-bit atomic per CTA (skipped if 0).
#include "tri_common.cuh"

namespace {

struct CollideArgs {
    const float4 *sph;
    int64_t n;
    uint64_t omega_begin, omega_end;
    int64_t tile_row_begin;
    unsigned long long *count;
};

typedef unsigned long long f2;   // packed f32x2 in a 64-bit register

__device__ __forceinline__ f2 pk(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk(f2 v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Exact scalar predicate (the ABI's operation order).
__device__ __forceinline__ uint32_t hit(const float4 a, float xj, float yj, float zj, float rj) {
    const float dx = __fsub_rn(a.x, xj);
    const float dy = __fsub_rn(a.y, yj);
    const float dz = __fsub_rn(a.z, zj);
    const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
    const float s = __fadd_rn(a.w, rj);
    return d2 < __fmul_rn(s, s) ? 1u : 0u;
}

// A' = |x|^2 - r^2 - kappa u (|x|^2 + r^2): the per-sphere part of the filter gap.
constexpr float kFilterKappaU = 64.0f / 16777216.0f;     // kappa u = 2^-18
__device__ __forceinline__ float filter_a(const float4 c) {
    const float q = fmaf(c.z, c.z, fmaf(c.y, c.y, c.x * c.x));
    const float w = c.w * c.w;
    return fmaf(-kFilterKappaU, q + w, q - w);
}

// filter gap for the two packed row spheres against one column sphere (column
// values pre-scaled by -2, column A' folded into the start of the chain)
__device__ __forceinline__ f2 gap2(f2 x, f2 y, f2 z, f2 r, f2 A, f2 cx, f2 cy, f2 cz, f2 cr, f2 cA) {
    return add2(A, fma2(x, cx, fma2(y, cy, fma2(z, cz, fma2(r, cr, cA)))));
}

__device__ __forceinline__ float4 load_sphere(const CollideArgs &a, int64_t idx) {
    if (idx < a.n) return __ldg(a.sph + idx);
    const float nan = __int_as_float(0x7fffffff);
    return make_float4(nan, nan, nan, nan);
}

// row spheres per thread
template <int RHO> constexpr int rows_per_thread() { return RHO >= 256 ? 8 : 4; }
constexpr int BLK = 32;       // columns per flag block

// column spheres, structure of arrays: -2x, -2y, -2z, -2r and A' (20 B per sphere);
// an aligned float4 of one array is two packed f32x2 operands (columns c, c+1 | c+2, c+3)
template <int RHO> struct ColSmemT { float v[5][RHO]; };

template <int RHO>
__device__ __forceinline__ uint32_t collide_tile(const CollideArgs &a, uint32_t bi, uint32_t bj, ColSmemT<RHO> &sm) {
    constexpr int K = rows_per_thread<RHO>();
    constexpr int NT = RHO / K;
    const int t = threadIdx.x;
    const int64_t r0 = (int64_t)bi * RHO, c0 = (int64_t)bj * RHO;
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const float4 c = load_sphere(a, c0 + t + q * NT);
        const int j = t + q * NT;
        sm.v[0][j] = -2.f * c.x; sm.v[1][j] = -2.f * c.y; sm.v[2][j] = -2.f * c.z; sm.v[3][j] = -2.f * c.w;
        sm.v[4][j] = filter_a(c);
    }
    float4 R[K];
#pragma unroll
    for (int q = 0; q < K; ++q) R[q] = load_sphere(a, r0 + t + q * NT);
    __syncthreads();
    uint32_t cnt = 0;
    auto recount = [&](int c, uint32_t strict_row_base) {
        const float xj = -0.5f * sm.v[0][c], yj = -0.5f * sm.v[1][c], zj = -0.5f * sm.v[2][c], rj = -0.5f * sm.v[3][c];
        uint32_t h = 0;
#pragma unroll
        for (int q = 0; q < K; ++q)
            h += ((uint32_t)c < strict_row_base + (uint32_t)(q * NT)) ? hit(R[q], xj, yj, zj, rj) : 0u;
        return h;
    };
    if (bi != bj) {
        f2 X[K], Y[K], Z[K], Q[K], A[K];                  // each row duplicated in both halves
#pragma unroll
        for (int k = 0; k < K; ++k) {
            X[k] = pk(R[k].x, R[k].x); Y[k] = pk(R[k].y, R[k].y); Z[k] = pk(R[k].z, R[k].z);
            Q[k] = pk(R[k].w, R[k].w);
            const float Ak = filter_a(R[k]);
            A[k] = pk(Ak, Ak);
        }
#pragma unroll 1
        for (int cb = 0; cb < RHO; cb += BLK) {
            uint32_t flags = 0;
#pragma unroll
            for (int c = 0; c < BLK; c += 4) {
                const float4 vx = *reinterpret_cast<const float4 *>(&sm.v[0][cb + c]);
                const float4 vy = *reinterpret_cast<const float4 *>(&sm.v[1][cb + c]);
                const float4 vz = *reinterpret_cast<const float4 *>(&sm.v[2][cb + c]);
                const float4 vr = *reinterpret_cast<const float4 *>(&sm.v[3][cb + c]);
                const float4 va = *reinterpret_cast<const float4 *>(&sm.v[4][cb + c]);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const f2 cx = h ? pk(vx.z, vx.w) : pk(vx.x, vx.y), cy = h ? pk(vy.z, vy.w) : pk(vy.x, vy.y);
                    const f2 cz = h ? pk(vz.z, vz.w) : pk(vz.x, vz.y), cr = h ? pk(vr.z, vr.w) : pk(vr.x, vr.y);
                    const f2 cA = h ? pk(va.z, va.w) : pk(va.x, va.y);
                    float mlo = __int_as_float(0x7f800000), mhi = mlo;
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        float glo, ghi;
                        upk(gap2(X[k], Y[k], Z[k], Q[k], A[k], cx, cy, cz, cr, cA), glo, ghi);
                        mlo = fminf(mlo, glo);
                        mhi = fminf(mhi, ghi);
                    }
                    flags |= (mlo < 0.f ? (1u << (c + 2 * h)) : 0u) | (mhi < 0.f ? (2u << (c + 2 * h)) : 0u);
                }
            }
            if (__any_sync(0xffffffffu, flags != 0)) {
#pragma unroll 1
                while (flags) {
                    const int c = __ffs(flags) - 1;
                    flags &= flags - 1;
                    cnt += recount(cb + c, 0xffffffffu - (uint32_t)(K * NT));
                }
            }
        }
    } else {  // diagonal tile: strict lower triangle, col < row (scalar, exact)
#pragma unroll 4
        for (int c = 0; c < RHO; ++c) cnt += recount(c, (uint32_t)t);
    }
    __syncthreads();  // smem reused by the next tile (persistent form)
    return cnt;
}

template <int NT>
__device__ __forceinline__ void flush_count(uint32_t cnt, unsigned long long *dst) {
    __shared__ uint32_t red[(NT + 31) / 32];
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
#pragma unroll
        for (int w = 0; w < (NT + 31) / 32; ++w) s += red[w];
        if (s) atomicAdd(dst, s);
    }
}

template <int RHO, int STRAT>
__global__ void __launch_bounds__(RHO / rows_per_thread<RHO>()) collide_kernel(CollideArgs a) {
    __shared__ __align__(16) ColSmemT<RHO> smem;
    uint32_t cnt = 0;
    if (STRAT == TRI_BB) {
        const uint32_t bj = blockIdx.x;
        const uint32_t bi = blockIdx.y + (uint32_t)a.tile_row_begin;
        if (bj > bi) return;
        cnt = collide_tile<RHO>(a, bi, bj, smem);
    } else if (STRAT == TRI_LAMBDA) {
        const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (w >= a.omega_end) return;
        uint32_t bi, bj;
        tri::lambda_map(w, bi, bj);
        cnt = collide_tile<RHO>(a, bi, bj, smem);
    } else {
#pragma unroll 1
        for (tri::TileWalk t(a.omega_begin, a.omega_end); t.more(); t.next())
            cnt += collide_tile<RHO>(a, t.bi, t.bj, smem);
    }
    flush_count<RHO / rows_per_thread<RHO>()>(cnt, a.count);
}


template <int RHO>
tri_status launch_r(const tri_map_t &m, int strategy, CollideArgs a, cudaStream_t st) {
    constexpr int NT = RHO / rows_per_thread<RHO>();
    if (strategy == TRI_BB) {
        const int64_t tr0 = m.row_begin / m.rho;
        const int64_t tr1 = (m.row_end + m.rho - 1) / m.rho;
        if (tr1 <= tr0) return TRI_OK;
        if (tr1 - tr0 > 65535) return TRI_ENOTSUP;
        a.tile_row_begin = tr0;
        collide_kernel<RHO, TRI_BB><<<dim3((unsigned)m.m, (unsigned)(tr1 - tr0)), NT, 0, st>>>(a);
    } else if (strategy == TRI_LAMBDA) {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        collide_kernel<RHO, TRI_LAMBDA><<<tri::tile_grid(nb), NT, 0, st>>>(a);
    } else {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, collide_kernel<RHO, TRI_LAMBDA_PERSIST>, NT, 0);
        uint64_t g = (uint64_t)tri::sm_count() * (uint64_t)(per_sm > 0 ? per_sm : 1);
        if (g > nb) g = nb;
        collide_kernel<RHO, TRI_LAMBDA_PERSIST><<<(unsigned)g, NT, 0, st>>>(a);
    }
    tri::note_launches(1);
    return tri::cuda_status();
}

}  // namespace

namespace tri {

tri_status launch_collide(const tri_map_t &m, int strategy, const float *sph, unsigned long long *count,
                          cudaStream_t st) {
    if (cudaMemsetAsync(count, 0, sizeof(unsigned long long), st) != cudaSuccess) return TRI_ECUDA;
    CollideArgs a;
    a.sph = (const float4 *)sph;
    a.n = m.n;
    a.omega_begin = m.omega_begin;
    a.omega_end = m.omega_end;
    a.tile_row_begin = 0;
    a.count = count;
    switch (m.rho) {
        case 128: return launch_r<128>(m, strategy, a, st);
        case 256: return launch_r<256>(m, strategy, a, st);
        default: return launch_r<512>(m, strategy, a, st);
    }
}

}  // namespace tri
