// Probe (not product code): does the EDM's gap to the write-only ceiling come from
// warp stores that straddle 128-byte lines?  Constant-value streaming stores over
// the packed lower triangle of n = 65536 fp32 cells (8.59 GB), four patterns:
//   0 linear sweep, each warp store = 512 B aligned to 128 B (fill_-like)
//   1 the same sweep shifted by 48 B (every warp store touches 5 lines, 2 partial)
//   2 EDM tiles (rho = 128, lambda grid, 8 warps, warp per row segment), 16-byte chunk
//     ownership: a row segment's store starts at the first 16-B boundary (today's kernel)
//   3 EDM tiles, 128-byte LINE ownership: a row segment's store starts at the first
//     128-B boundary in the segment, so every warp store is 4 whole lines
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void st4(float *p, float v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(p), "f"(v) : "memory");
}

__global__ void lin(float *out, uint64_t cells, int shift_floats) {
    const uint64_t nchunks = (cells - 64) / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += stride)
        st4(out + shift_floats + 4 * c, 1.f);
}

__host__ __device__ __forceinline__ uint64_t T2(uint64_t r) { return r * (r + 1) / 2; }

__device__ __forceinline__ void lam(uint64_t w, uint32_t &bi, uint32_t &bj) {
    float x = 8.f * (float)w + 1.f;
    uint64_t i = (uint64_t)((sqrtf(x) - 1.f) * 0.5f);
    while (T2(i) > w) --i;
    while (T2(i + 1) <= w) ++i;
    bi = (uint32_t)i; bj = (uint32_t)(w - T2(i));
}

template <int ALIGN>   // floats: 4 (16 B) or 32 (128 B)
__global__ void __launch_bounds__(256) tiles(float *out, int64_t n) {
    uint32_t bi, bj;
    lam(blockIdx.x, bi, bj);
    if (bj + 1 >= bi) return;                  // interior tiles only (99 % of the cells)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)bi * 128 + warp * 16, c0 = (int64_t)bj * 128;
    uint64_t s = T2(r0) + c0;
#pragma unroll 1
    for (int rr = 0; rr < 16; ++rr) {
        const int delta = (int)((0u - (uint32_t)s) & (ALIGN - 1));
        st4(out + s + delta + 4 * lane, 1.f);
        s += (uint64_t)(r0 + rr + 1);
    }
}

extern "C" int run_probe(int which, float *out, int64_t n, int grid, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t cells = T2((uint64_t)n);
    const uint32_t tilesN = (uint32_t)T2((uint64_t)(n / 128));
    switch (which) {
    case 0: lin<<<grid, 256, 0, st>>>(out, cells, 0); break;
    case 1: lin<<<grid, 256, 0, st>>>(out, cells, 12); break;
    case 2: tiles<4><<<tilesN, 256, 0, st>>>(out, n); break;
    case 3: tiles<32><<<tilesN, 256, 0, st>>>(out, n); break;
    }
    return (int)cudaGetLastError();
}
