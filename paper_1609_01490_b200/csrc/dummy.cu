// dummy.cu -- the paper's map-cost "dummy kernel".
//
// One thread per cell, rho x rho threads per CTA: every thread
// obtains its tile coordinate -- lambda(omega) (Eq. 4) for TRI_LAMBDA /
// TRI_LAMBDA_PERSIST, the identity + block discard for TRI_BB --
// adds its local offset (block-space mapping), filters j <= i < n
// and performs the mode's memory action.  The kernel exists to measure the
// map's cost, so the per-thread work is deliberately minimal.
#include "tri_common.cuh"

namespace {

struct DummyArgs {
    int64_t n;
    uint64_t omega_begin, omega_end;  // lambda tiles
    int64_t tile_row_begin;           // BB: first tile row (grid.y offset)
    uint64_t out_offset;
    void *out;
    int wide;                         // PACKED element: 0 = u32, 1 = u64
    int strict;                       // diag = 0: keep j < i only
};

template <int RHO, int MODE>
__device__ __forceinline__ void dummy_body(const DummyArgs &a, uint32_t bi, uint32_t bj,
                                           unsigned long long *acc) {
    const int64_t i = (int64_t)bi * RHO + threadIdx.y;
    const int64_t j = (int64_t)bj * RHO + threadIdx.x;
    const bool ok = (i < a.n) && (a.strict ? j < i : j <= i);
    if (MODE == TRI_DUMMY_FIXED) {
        if (ok) *(volatile uint32_t *)a.out = (uint32_t)(i + j);
    } else if (MODE == TRI_DUMMY_PACKED) {
        if (ok) {
            const uint64_t idx = tri::T2((uint64_t)i) + (uint64_t)j - a.out_offset;
            if (a.wide)
                ((unsigned long long *)a.out)[idx] = ((unsigned long long)i << 32) | (unsigned long long)j;
            else
                ((uint32_t *)a.out)[idx] = ((uint32_t)i << 16) | (uint32_t)j;
        }
    } else if (MODE == TRI_DUMMY_DIGEST) {
        *acc += ok ? (unsigned long long)(i + j) : 0ull;
    } else {  // COUNT
        *acc += ok ? 1ull : 0ull;
    }
}

// Block reduction of a per-thread u64; the total is returned to thread (0,0).
template <int NT>
__device__ __forceinline__ unsigned long long block_sum(unsigned long long v) {
    __shared__ unsigned long long red[NT / 32];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int t = threadIdx.y * blockDim.x + threadIdx.x;
    if ((t & 31) == 0) red[t >> 5] = v;
    __syncthreads();
    unsigned long long s = 0;
    if (t == 0)
        for (int w = 0; w < NT / 32; ++w) s += red[w];
    return s;
}

template <int RHO, int MODE, int STRAT>
__global__ void __launch_bounds__(RHO * RHO) dummy_kernel(DummyArgs a) {
    unsigned long long acc = 0;
    unsigned long long *cnt = (unsigned long long *)a.out;
    if (STRAT == TRI_BB) {
        const uint32_t bj = blockIdx.x;
        const uint32_t bi = blockIdx.y + (uint32_t)a.tile_row_begin;
        if (bj > bi) {                                   // tile above the diagonal: discard
            if (MODE == TRI_DUMMY_COUNT && threadIdx.x == 0 && threadIdx.y == 0) {
                atomicAdd(&cnt[0], 1ull);
                atomicAdd(&cnt[1], 1ull);
                atomicAdd(&cnt[2], (unsigned long long)(RHO * RHO));
                atomicAdd(&cnt[4], (unsigned long long)(RHO * RHO));
            }
            return;
        }
        dummy_body<RHO, MODE>(a, bi, bj, &acc);
    } else if (STRAT == TRI_LAMBDA) {
        const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (w >= a.omega_end) return;                    // 2-D grid tail (only when B >= 2^30)
        uint32_t bi, bj;
        tri::lambda_map(w, bi, bj);
        dummy_body<RHO, MODE>(a, bi, bj, &acc);
    } else if (STRAT >= TRI_LAMBDA_X) {
        // the paper's uncorrected sqrt variants (section 4.1): outside their
        // validity range the tile is wrong; tiles outside the triangle are skipped
        const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (w >= a.omega_end) return;
        uint32_t bi, bj;
        tri::lambda_variant(w, STRAT - TRI_LAMBDA_X + TRI_SQRT_X, bi, bj);
        if (bj > bi || (int64_t)bi * RHO >= a.n) return;
        dummy_body<RHO, MODE>(a, bi, bj, &acc);
    } else {  // persistent lambda-walk
        for (tri::TileWalk t(a.omega_begin, a.omega_end); t.more(); t.next()) dummy_body<RHO, MODE>(a, t.bi, t.bj, &acc);
    }
    if (MODE == TRI_DUMMY_DIGEST) {
        const unsigned long long s = block_sum<RHO * RHO>(acc);
        if (threadIdx.x == 0 && threadIdx.y == 0 && s) atomicAdd(cnt, s);
    } else if (MODE == TRI_DUMMY_COUNT) {
        const unsigned long long useful = block_sum<RHO * RHO>(acc);
        if (threadIdx.x == 0 && threadIdx.y == 0) {
            unsigned long long tiles = 1;
            if (STRAT == TRI_LAMBDA_PERSIST) {
                const tri::TileWalk t(a.omega_begin, a.omega_end);
                tiles = t.end - t.w;
            }
            atomicAdd(&cnt[0], tiles);
            atomicAdd(&cnt[2], tiles * RHO * RHO);
            atomicAdd(&cnt[3], useful);
            atomicAdd(&cnt[4], tiles * RHO * RHO - useful);
        }
    }
}

template <int RHO, int MODE>
tri_status launch3(const tri_map_t &m, int strategy, DummyArgs a, cudaStream_t st) {
    const dim3 blk(RHO, RHO);
    if (strategy == TRI_BB) {
        const int64_t tr0 = m.row_begin / m.rho;
        const int64_t tr1 = (m.row_end + m.rho - 1) / m.rho;
        if (tr1 <= tr0) return TRI_OK;
        if (m.m > 0x7fffffffll || tr1 - tr0 > 65535) return TRI_ENOTSUP;
        a.tile_row_begin = tr0;
        dummy_kernel<RHO, MODE, TRI_BB><<<dim3((unsigned)m.m, (unsigned)(tr1 - tr0)), blk, 0, st>>>(a);
    } else if (strategy == TRI_LAMBDA) {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        dummy_kernel<RHO, MODE, TRI_LAMBDA><<<tri::tile_grid(nb), blk, 0, st>>>(a);
    } else if (strategy >= TRI_LAMBDA_X) {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        if (strategy == TRI_LAMBDA_X)
            dummy_kernel<RHO, MODE, TRI_LAMBDA_X><<<tri::tile_grid(nb), blk, 0, st>>>(a);
        else if (strategy == TRI_LAMBDA_N)
            dummy_kernel<RHO, MODE, TRI_LAMBDA_N><<<tri::tile_grid(nb), blk, 0, st>>>(a);
        else
            dummy_kernel<RHO, MODE, TRI_LAMBDA_R><<<tri::tile_grid(nb), blk, 0, st>>>(a);
    } else {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dummy_kernel<RHO, MODE, TRI_LAMBDA_PERSIST>,
                                                      RHO * RHO, 0);
        uint64_t g = (uint64_t)tri::sm_count() * (uint64_t)(per_sm > 0 ? per_sm : 1);
        if (g > nb) g = nb;
        dummy_kernel<RHO, MODE, TRI_LAMBDA_PERSIST><<<(unsigned)g, blk, 0, st>>>(a);
    }
    tri::note_launches(1);
    return tri::cuda_status();
}

template <int RHO>
tri_status launch2(const tri_map_t &m, int strategy, int mode, DummyArgs a, cudaStream_t st) {
    switch (mode) {
        case TRI_DUMMY_FIXED: return launch3<RHO, TRI_DUMMY_FIXED>(m, strategy, a, st);
        case TRI_DUMMY_PACKED: return launch3<RHO, TRI_DUMMY_PACKED>(m, strategy, a, st);
        case TRI_DUMMY_DIGEST: return launch3<RHO, TRI_DUMMY_DIGEST>(m, strategy, a, st);
        default: return launch3<RHO, TRI_DUMMY_COUNT>(m, strategy, a, st);
    }
}

}  // namespace

namespace tri {

tri_status launch_dummy(const tri_map_t &m, int strategy, int mode, void *d_out, cudaStream_t st) {
    if (mode == TRI_DUMMY_DIGEST || mode == TRI_DUMMY_COUNT) {
        if (cudaMemsetAsync(d_out, 0, mode == TRI_DUMMY_DIGEST ? 8 : 40, st) != cudaSuccess)
            return TRI_ECUDA;
    }
    DummyArgs a;
    a.n = m.n;
    a.omega_begin = m.omega_begin;
    a.omega_end = m.omega_end;
    a.tile_row_begin = 0;
    a.out_offset = m.out_offset;
    a.out = d_out;
    a.wide = m.n > 65536 ? 1 : 0;
    a.strict = m.diag ? 0 : 1;
    switch (m.rho) {
        case 8: return launch2<8>(m, strategy, mode, a, st);
        case 16: return launch2<16>(m, strategy, mode, a, st);
        default: return launch2<32>(m, strategy, mode, a, st);
    }
}

}  // namespace tri
