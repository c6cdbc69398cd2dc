// collide1d.cu -- 1-D collision count ("collision
// detection in 1D/3D"; reading Q10: intervals [c - r, c + r] on [0, 1)).
//
// Pairs j < i with |c_i - c_j| < r_i + r_j, evaluated in IEEE fp32 as
//   d = ci - cj;  s = ri + rj;  |d| < s
// (fp32 subtraction |d| - s is sign-exact without FTZ, so the hot loop keeps
// min(|d| - s) per 32-column block and recounts blocks with a negative minimum
// with the predicate itself, as in collide.cu).
//
// Tiles of rho x rho intervals.  The lambda strategy launches the T(m-1)
// strictly-lower tiles through Eq. 5 (lambda_nodiag, corrected),
// which need no per-pair filter, followed by the m diagonal tiles, which apply
// the strict filter j < i -- one launch, B = T(m-1) + m = T(m) CTAs.  BB: the
// m x m grid with tiles above the diagonal discarded.
#include "tri_common.cuh"

namespace {

struct C1Args {
    const float2 *iv;       // (centre, radius)
    int64_t n;
    uint64_t omega_begin, omega_end;
    uint64_t offdiag;       // T(m-1): tiles below the diagonal
    int64_t tile_row_begin;
    unsigned long long *count;
};

constexpr int NT = 128;
constexpr int K = 2;        // row intervals per thread
constexpr int RHO = NT * K; // 256
constexpr int BLK = 32;

__device__ __forceinline__ uint32_t hit1(const float2 a, const float2 b) {
    const float d = __fsub_rn(a.x, b.x);
    const float s = __fadd_rn(a.y, b.y);
    return fabsf(d) < s ? 1u : 0u;
}

__device__ __forceinline__ float2 load_iv(const C1Args &a, int64_t idx) {
    if (idx < a.n) return __ldg(a.iv + idx);
    const float nan = __int_as_float(0x7fffffff);
    return make_float2(nan, nan);
}

__device__ __forceinline__ uint32_t tile(const C1Args &a, uint32_t bi, uint32_t bj, float2 *sm) {
    const int t = threadIdx.x;
    const int64_t r0 = (int64_t)bi * RHO, c0 = (int64_t)bj * RHO;
    sm[t] = load_iv(a, c0 + t);
    sm[t + NT] = load_iv(a, c0 + t + NT);
    const float2 A = load_iv(a, r0 + t), B = load_iv(a, r0 + t + NT);
    __syncthreads();
    uint32_t cnt = 0;
    if (bi != bj) {
#pragma unroll 1
        for (int cb = 0; cb < RHO; cb += BLK) {
            float m = __int_as_float(0x7f800000);
#pragma unroll 8
            for (int c = cb; c < cb + BLK; ++c) {
                const float2 v = sm[c];
                const float ga = __fsub_rn(fabsf(__fsub_rn(A.x, v.x)), __fadd_rn(A.y, v.y));
                const float gb = __fsub_rn(fabsf(__fsub_rn(B.x, v.x)), __fadd_rn(B.y, v.y));
                m = fminf(m, fminf(ga, gb));
            }
            if (__any_sync(0xffffffffu, m < 0.f)) {
                if (m < 0.f)
                    for (int c = cb; c < cb + BLK; ++c) cnt += hit1(A, sm[c]) + hit1(B, sm[c]);
            }
        }
    } else {                                        // diagonal tile: strict j < i
#pragma unroll 4
        for (int c = 0; c < RHO; ++c) {
            const float2 v = sm[c];
            cnt += (c < t) ? hit1(A, v) : 0u;
            cnt += (c < t + NT) ? hit1(B, v) : 0u;
        }
    }
    __syncthreads();
    return cnt;
}

template <int STRAT>
__global__ void __launch_bounds__(NT) collide1d_kernel(C1Args a) {
    __shared__ float2 sm[RHO];
    __shared__ uint32_t red[NT / 32];
    uint32_t cnt = 0;
    if (STRAT == TRI_BB) {
        const uint32_t bj = blockIdx.x, bi = blockIdx.y + (uint32_t)a.tile_row_begin;
        if (bj > bi) return;
        cnt = tile(a, bi, bj, sm);
    } else {
        const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (w >= a.omega_end) return;
        uint32_t bi, bj;
        if (w < a.offdiag) tri::lambda_nodiag(w, bi, bj);           // Eq. 5: strictly below
        else bi = bj = (uint32_t)(w - a.offdiag);                    // the diagonal tiles
        cnt = tile(a, bi, bj, sm);
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < NT / 32; ++w) s += red[w];
        if (s) atomicAdd(a.count, s);
    }
}

}  // namespace

namespace tri {

// Whole-domain (world = 1) or snapped-row ranks for BB; lambda splits its
// T(m) tiles (off-diagonal first) evenly by the map's plain omega range.
tri_status launch_collide1d(const tri_map_t &m, int strategy, const float *iv, unsigned long long *count,
                            cudaStream_t st) {
    if (cudaMemsetAsync(count, 0, sizeof(unsigned long long), st) != cudaSuccess) return TRI_ECUDA;
    C1Args a;
    a.iv = (const float2 *)iv;
    a.n = m.n;
    a.offdiag = T2((uint64_t)m.m - 1);
    a.count = count;
    a.tile_row_begin = 0;
    a.omega_begin = (uint64_t)(((unsigned __int128)m.rank * m.blocks) / (uint64_t)m.world);
    a.omega_end = (uint64_t)(((unsigned __int128)(m.rank + 1) * m.blocks) / (uint64_t)m.world);
    if (strategy == TRI_BB) {
        const int64_t tr0 = m.row_begin / m.rho, tr1 = (m.row_end + m.rho - 1) / m.rho;
        if (tr1 <= tr0) return TRI_OK;
        if (tr1 - tr0 > 65535) return TRI_ENOTSUP;
        a.tile_row_begin = tr0;
        collide1d_kernel<TRI_BB><<<dim3((unsigned)m.m, (unsigned)(tr1 - tr0)), NT, 0, st>>>(a);
    } else {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        collide1d_kernel<TRI_LAMBDA><<<tile_grid(nb), NT, 0, st>>>(a);
    }
    note_launches(1);
    return cuda_status();
}

}  // namespace tri
