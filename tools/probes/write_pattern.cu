// Probe (not product code): pure streaming stores over the packed lower
// triangle of n = 65536 fp32 cells (8.59 GB), to locate the EDM's gap to the
// write-only ceiling.  Warp w writes rows w, w + W, ... contiguously, with
// 16-byte (st.global.v4) or 32-byte (st.global.v8, sm_100) stores per lane.
#include <cstdint>
#include <cuda_runtime.h>
template <int V>
__global__ void probe_rows(float *out, int64_t n) {
    const int64_t W = (int64_t)gridDim.x * blockDim.x / 32;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    for (int64_t r = w; r < n; r += W) {
        const int64_t a = (r * (r + 1) / 2) / V, b = ((r + 1) * (r + 2) / 2 + V - 1) / V;   // V-float units
        for (int64_t c = a + lane; c < b; c += 32) {
            float *p = out + c * V;
            if (V == 4)
                asm volatile("st.global.cs.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(p), "f"(1.f) : "memory");
            else
                asm volatile("st.global.cs.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "f"(1.f) : "memory");
        }
    }
}
extern "C" int run_probe(int which, float *out, int64_t n, int grid, int block, void *stream) {
    if (which == 0) probe_rows<4><<<grid, block, 0, (cudaStream_t)stream>>>(out, n);
    else probe_rows<8><<<grid, block, 0, (cudaStream_t)stream>>>(out, n);
    return (int)cudaGetLastError();
}
