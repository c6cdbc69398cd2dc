// rb.cu -- the RB (rectangular box) comparator map (reading Q19)
// for the dummy kernel and the EDM: the paper's fastest strategy for global
// memory on Kepler, built here as a third comparator beside lambda
// and BB.  One thread per cell of the H x W folded rectangle (tri::rb_map);
// consecutive threads in x map to consecutive columns of one triangle row, so
// the per-cell stores of a warp are contiguous except at the fold.
#include "tri_common.cuh"

namespace {

struct RbArgs {
    int64_t n;
    void *out;
    int wide;
    const float *pts;
    int64_t ld;
};

template <int RHO, int MODE>
__global__ void __launch_bounds__(RHO * RHO) dummy_rb_kernel(RbArgs a) {
    const int64_t x = (int64_t)blockIdx.x * RHO + threadIdx.x;
    const int64_t y = (int64_t)blockIdx.y * RHO + threadIdx.y;
    int64_t i = 0, j = 0;
    const bool ok = tri::rb_map(x, y, a.n, i, j);
    unsigned long long *cnt = (unsigned long long *)a.out;
    unsigned long long acc = 0;
    if (MODE == TRI_DUMMY_FIXED) {
        if (ok) *(volatile uint32_t *)a.out = (uint32_t)(i + j);
    } else if (MODE == TRI_DUMMY_PACKED) {
        if (ok) {
            const uint64_t idx = tri::T2((uint64_t)i) + (uint64_t)j;
            if (a.wide)
                ((unsigned long long *)a.out)[idx] = ((unsigned long long)i << 32) | (unsigned long long)j;
            else
                ((uint32_t *)a.out)[idx] = ((uint32_t)i << 16) | (uint32_t)j;
        }
    } else {
        acc = ok ? (MODE == TRI_DUMMY_DIGEST ? (unsigned long long)(i + j) : 1ull) : 0ull;
        __shared__ unsigned long long red[RHO * RHO / 32];
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const int t = threadIdx.y * RHO + threadIdx.x;
        if ((t & 31) == 0) red[t >> 5] = acc;
        __syncthreads();
        if (t == 0) {
            unsigned long long s = 0;
            for (int w = 0; w < RHO * RHO / 32; ++w) s += red[w];
            if (MODE == TRI_DUMMY_DIGEST) {
                if (s) atomicAdd(cnt, s);
            } else {
                atomicAdd(&cnt[0], 1ull);
                atomicAdd(&cnt[2], (unsigned long long)(RHO * RHO));
                atomicAdd(&cnt[3], s);
                atomicAdd(&cnt[4], (unsigned long long)(RHO * RHO) - s);
            }
        }
    }
}

// EDM under RB: one cell per thread, blocks of 32 x 8 threads (x = columns).
template <int DIM>
__global__ void __launch_bounds__(256) edm_rb_kernel(RbArgs a) {
    const int64_t x = (int64_t)blockIdx.x * 32 + threadIdx.x;
    const int64_t y = (int64_t)blockIdx.y * 8 + threadIdx.y;
    int64_t i, j;
    if (!tri::rb_map(x, y, a.n, i, j)) return;
    float d2 = 0.f;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
        const float dd = __ldg(a.pts + i * a.ld + d) - __ldg(a.pts + j * a.ld + d);
        d2 = d == 0 ? dd * dd : fmaf(dd, dd, d2);
    }
    ((float *)a.out)[tri::T2((uint64_t)i) + (uint64_t)j] = sqrt_approx(d2);
}

inline void rect(int64_t n, int64_t &H, int64_t &W) {
    const int64_t h = n / 2;
    H = n - h;
    W = 2 * h + 1;
}

template <int RHO>
tri_status dummy_rb(int64_t n, int mode, RbArgs a, cudaStream_t st) {
    int64_t H, W;
    rect(n, H, W);
    const dim3 grid((unsigned)((W + RHO - 1) / RHO), (unsigned)((H + RHO - 1) / RHO));
    if ((W + RHO - 1) / RHO > 0x7fffffff || (H + RHO - 1) / RHO > 65535) return TRI_ENOTSUP;
    const dim3 blk(RHO, RHO);
    switch (mode) {
        case TRI_DUMMY_FIXED: dummy_rb_kernel<RHO, TRI_DUMMY_FIXED><<<grid, blk, 0, st>>>(a); break;
        case TRI_DUMMY_PACKED: dummy_rb_kernel<RHO, TRI_DUMMY_PACKED><<<grid, blk, 0, st>>>(a); break;
        case TRI_DUMMY_DIGEST: dummy_rb_kernel<RHO, TRI_DUMMY_DIGEST><<<grid, blk, 0, st>>>(a); break;
        default: dummy_rb_kernel<RHO, TRI_DUMMY_COUNT><<<grid, blk, 0, st>>>(a); break;
    }
    tri::note_launches(1);
    return tri::cuda_status();
}

}  // namespace

namespace tri {

tri_status launch_dummy_rb(const tri_map_t &m, int mode, void *d_out, cudaStream_t st) {
    if (m.world > 1) return TRI_ENOTSUP;
    if (mode == TRI_DUMMY_DIGEST || mode == TRI_DUMMY_COUNT) {
        if (cudaMemsetAsync(d_out, 0, mode == TRI_DUMMY_DIGEST ? 8 : 40, st) != cudaSuccess) return TRI_ECUDA;
    }
    RbArgs a;
    a.n = m.n;
    a.out = d_out;
    a.wide = m.n > 65536 ? 1 : 0;
    a.pts = nullptr;
    a.ld = 0;
    switch (m.rho) {
        case 8: return dummy_rb<8>(m.n, mode, a, st);
        case 16: return dummy_rb<16>(m.n, mode, a, st);
        default: return dummy_rb<32>(m.n, mode, a, st);
    }
}

tri_status launch_edm_rb(const tri_map_t &m, const float *pts, int dim, int64_t ld, float *out, cudaStream_t st) {
    if (m.world > 1) return TRI_ENOTSUP;
    int64_t H, W;
    rect(m.n, H, W);
    if ((H + 7) / 8 > 65535) return TRI_ENOTSUP;
    RbArgs a;
    a.n = m.n;
    a.out = out;
    a.wide = 0;
    a.pts = pts;
    a.ld = ld;
    const dim3 grid((unsigned)((W + 31) / 32), (unsigned)((H + 7) / 8)), blk(32, 8);
    switch (dim) {
        case 1: edm_rb_kernel<1><<<grid, blk, 0, st>>>(a); break;
        case 2: edm_rb_kernel<2><<<grid, blk, 0, st>>>(a); break;
        case 3: edm_rb_kernel<3><<<grid, blk, 0, st>>>(a); break;
        default: edm_rb_kernel<4><<<grid, blk, 0, st>>>(a); break;
    }
    note_launches(1);
    return cuda_status();
}

}  // namespace tri
