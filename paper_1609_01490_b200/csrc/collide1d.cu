// collide1d.cu -- 1-D collision count ("collision
// detection in 1D/3D"; reading Q10: intervals [c - r, c + r] on [0, 1)).
//
// Pairs j < i with |c_i - c_j| < r_i + r_j, evaluated in IEEE fp32 as
//   d = ci - cj;  s = ri + rj;  |d| < s
// The hot loop only FILTERS, on interval end points widened by a rounding
// margin: lo' = (c - r) - M, hi' = (c + r) + M, M = kappa u (|c| + r) (u = 2^-24,
// kappa = 8).  With S = |c| + r: a pair the predicate counts has
// (ci - cj) - (ri + rj) < 2.01 u (ri + rj) (first order; likewise cj - ci),
// while fl(lo'_i) <= ci - ri - M_i + 2u S_i and fl(hi'_j) >= cj + rj + M_j - 2u S_j,
// so lo'_i - hi'_j < (4.01 - kappa (1 - 3u)) u (S_i + S_j) < 0 for kappa > 4.02;
// the same for lo'_j - hi'_i.  With the row stored as (lo'_i, -hi'_i) and the
// column as (-hi'_j, lo'_j), ONE packed FADD2 gives both differences (their
// signs are exact: rounding preserves sign), and one LOP3 folds
// acc |= g1 & g2 (sign bits: "both negative" for some pair).  Blocks whose
// accumulator has the sign bit set are re-filtered pair by pair and the
// flagged pairs counted with the predicate itself, so the count is exact.
// (NaN padding is the positive canonical NaN: never flags; -0 only flags.)
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

constexpr int NT = 64;
constexpr int K = 4;        // row intervals per thread (one column load serves 4 x 32 pairs)
constexpr int RHO = NT * K; // 256
constexpr int BLK = 8;     // columns per flag block: at ~2e-5 hits per pair a warp's 4 x 32 x BLK
                           // pairs flag ~2 % of blocks, each re-filtered at ~2x the block's cost
constexpr float kMarginKappaU = 8.0f / 16777216.0f;     // kappa u = 2^-21 (the bound needs kappa > 4.02)

typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint32_t lop3_or_and(uint32_t acc, uint32_t x, uint32_t y) {  // acc | (x & y)
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xf8;" : "=r"(d) : "r"(acc), "r"(x), "r"(y));
    return d;
}
// widened end points (lo', hi') of one interval
__device__ __forceinline__ float2 ends(const float2 v) {
    const float M = kMarginKappaU * (fabsf(v.x) + v.y);
    return make_float2(__fsub_rn(__fsub_rn(v.x, v.y), M), __fadd_rn(__fadd_rn(v.x, v.y), M));
}

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

__device__ __forceinline__ uint32_t tile(const C1Args &a, uint32_t bi, uint32_t bj, float2 *sm, float2 *sf) {
    const int t = threadIdx.x;
    const int64_t r0 = (int64_t)bi * RHO, c0 = (int64_t)bj * RHO;
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const float2 v = load_iv(a, c0 + t + q * NT);
        const float2 e = ends(v);
        sm[t + q * NT] = v;                               // (c, r): the exact predicate
        sf[t + q * NT] = make_float2(-e.y, e.x);          // (-hi', lo'): the filter
    }
    float2 R[K];
#pragma unroll
    for (int q = 0; q < K; ++q) R[q] = load_iv(a, r0 + t + q * NT);
    __syncthreads();
    uint32_t cnt = 0;
    if (bi != bj) {
        f2 E[K];
#pragma unroll
        for (int q = 0; q < K; ++q) {
            const float2 e = ends(R[q]);
            E[q] = pk(e.x, -e.y);                         // (lo'_i, -hi'_i)
        }
#pragma unroll 1
        for (int cb = 0; cb < RHO; cb += BLK) {
            uint32_t accq[K];                             // one chain per row (no serial LOP3 chain)
#pragma unroll
            for (int q = 0; q < K; ++q) accq[q] = 0;
#pragma unroll
            for (int c = cb; c < cb + BLK; ++c) {
                const float2 w = sf[c];
                const f2 cw = pk(w.x, w.y);
#pragma unroll
                for (int q = 0; q < K; ++q) {
                    const f2 g = add2(E[q], cw);          // (lo'_i - hi'_j, lo'_j - hi'_i)
                    accq[q] = lop3_or_and(accq[q], (uint32_t)g, (uint32_t)(g >> 32));
                }
            }
            uint32_t acc = 0;
#pragma unroll
            for (int q = 0; q < K; ++q) acc |= accq[q];
            if (__any_sync(0xffffffffu, (int32_t)acc < 0)) {
                if ((int32_t)acc < 0) {                   // rare: re-filter per pair, count exactly
#pragma unroll 1
                    for (int c = cb; c < cb + BLK; ++c) {
                        const float2 w = sf[c];
                        const f2 cw = pk(w.x, w.y);
#pragma unroll
                        for (int q = 0; q < K; ++q) {
                            const f2 g = add2(E[q], cw);
                            if ((int32_t)((uint32_t)g & (uint32_t)(g >> 32)) < 0) cnt += hit1(R[q], sm[c]);
                        }
                    }
                }
            }
        }
    } else {                                        // diagonal tile: strict j < i
#pragma unroll 4
        for (int c = 0; c < RHO; ++c) {
            const float2 v = sm[c];
#pragma unroll
            for (int q = 0; q < K; ++q) cnt += (c < t + q * NT) ? hit1(R[q], v) : 0u;
        }
    }
    __syncthreads();
    return cnt;
}

template <int STRAT>
__global__ void __launch_bounds__(NT) collide1d_kernel(C1Args a) {
    __shared__ float2 sm[RHO], sf[RHO];
    __shared__ uint32_t red[NT / 32];
    uint32_t cnt = 0;
    if (STRAT == TRI_BB) {
        const uint32_t bj = blockIdx.x, bi = blockIdx.y + (uint32_t)a.tile_row_begin;
        if (bj > bi) return;
        cnt = tile(a, bi, bj, sm, sf);
    } else {
        const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (w >= a.omega_end) return;
        uint32_t bi, bj;
        if (w < a.offdiag) tri::lambda_nodiag(w, bi, bj);           // Eq. 5: strictly below
        else bi = bj = (uint32_t)(w - a.offdiag);                    // the diagonal tiles
        cnt = tile(a, bi, bj, sm, sf);
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
