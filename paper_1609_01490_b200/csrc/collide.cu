// collide.cu -- all-pairs sphere collision count over the strict lower
// triangle ("collision detection of N spheres with random
// radius inside a unit box ... using a shared memory approach").
//
// Tile = rho x rho sphere pairs, coordinate from lambda(omega) or the BB grid.
// The rho column spheres of the tile are staged in shared memory (one float4
// each, read back as a warp-broadcast LDS.128); each of the rho/2 threads holds
// K = 2 row spheres in registers and tests them against every column sphere.
// The predicate is evaluated with explicit round-to-nearest intrinsics in
// exactly the order the ABI (include/tri.h) fixes, so the integer count is
// reproducible bit for bit:
//   dx = xi - xj, dy, dz;  d2 = fma(dz,dz, fma(dy,dy, dx*dx));  s = ri + rj;  d2 < s*s
// Out-of-range spheres are NaN (every comparison false).  Diagonal tiles add
// the strict filter col < row; other tiles run the unmasked loop.  Counts are
// reduced per warp, per CTA, then one 64-bit atomic per CTA (skipped if 0).
#include "tri_common.cuh"

namespace {

struct CollideArgs {
    const float4 *sph;
    int64_t n;
    uint64_t omega_begin, omega_end;
    int64_t tile_row_begin;
    unsigned long long *count;
};

__device__ __forceinline__ uint32_t hit(float xi, float yi, float zi, float ri, const float4 c) {
    const float dx = __fsub_rn(xi, c.x);
    const float dy = __fsub_rn(yi, c.y);
    const float dz = __fsub_rn(zi, c.z);
    const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
    const float s = __fadd_rn(ri, c.w);
    return d2 < __fmul_rn(s, s) ? 1u : 0u;
}

__device__ __forceinline__ float4 load_sphere(const CollideArgs &a, int64_t idx) {
    if (idx < a.n) return __ldg(a.sph + idx);
    const float nan = __int_as_float(0x7fffffff);
    return make_float4(nan, nan, nan, nan);
}

template <int RHO>
__device__ __forceinline__ uint32_t collide_tile(const CollideArgs &a, uint32_t bi, uint32_t bj,
                                                 float4 *smem) {
    constexpr int NT = RHO / 2;
    const int t = threadIdx.x;
    const int64_t r0 = (int64_t)bi * RHO, c0 = (int64_t)bj * RHO;
    smem[t] = load_sphere(a, c0 + t);
    smem[t + NT] = load_sphere(a, c0 + t + NT);
    const float4 A = load_sphere(a, r0 + t);
    const float4 B = load_sphere(a, r0 + t + NT);
    __syncthreads();
    uint32_t cnt = 0;
    if (bi != bj) {
#pragma unroll 8
        for (int c = 0; c < RHO; ++c) {
            const float4 s = smem[c];
            cnt += hit(A.x, A.y, A.z, A.w, s);
            cnt += hit(B.x, B.y, B.z, B.w, s);
        }
    } else {  // diagonal tile: strict lower triangle, col < row
#pragma unroll 8
        for (int c = 0; c < RHO; ++c) {
            const float4 s = smem[c];
            cnt += (c < t) ? hit(A.x, A.y, A.z, A.w, s) : 0u;
            cnt += (c < t + NT) ? hit(B.x, B.y, B.z, B.w, s) : 0u;
        }
    }
    __syncthreads();  // smem reused by the next tile (persistent form)
    return cnt;
}

template <int NT>
__device__ __forceinline__ void flush_count(uint32_t cnt, unsigned long long *dst) {
    __shared__ uint32_t red[NT / 32];
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) s += red[w];
        if (s) atomicAdd(dst, s);
    }
}

template <int RHO, int STRAT>
__global__ void __launch_bounds__(RHO / 2) collide_kernel(CollideArgs a) {
    __shared__ float4 smem[RHO];
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
        for (uint64_t w = a.omega_begin + blockIdx.x; w < a.omega_end; w += gridDim.x) {
            uint32_t bi, bj;
            tri::lambda_map(w, bi, bj);
            cnt += collide_tile<RHO>(a, bi, bj, smem);
        }
    }
    flush_count<RHO / 2>(cnt, a.count);
}

template <int RHO>
tri_status launch_r(const tri_map_t &m, int strategy, CollideArgs a, cudaStream_t st) {
    constexpr int NT = RHO / 2;
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
        case 64: return launch_r<64>(m, strategy, a, st);
        case 128: return launch_r<128>(m, strategy, a, st);
        default: return launch_r<256>(m, strategy, a, st);
    }
}

}  // namespace tri
