// Probe (tools only): tcgen05.ld throughput.  Each warp re-reads 128 columns of its TMEM lane
// quarter (32x32b shape) `iters` times with `inflight` loads outstanding, touching only
// one register per load (no ALU work).  One CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o _ab/libtmembw.so tools/probes/tmem_bw.cu
#include <cstdint>
#include <cuda_runtime.h>

#define LD32(v, addr)                                                                                              \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
                 "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                               \
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),   \
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),         \
                   "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),       \
                   "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),       \
                   "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                                         \
                 : "r"(addr))

#define LD16P(v, addr)                                                                                             \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),   \
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),         \
                   "=r"(v[15])                                                                                    \
                 : "r"(addr))

template <int kIn, bool kPack>
__global__ void __launch_bounds__(512, 1) bw(int iters, long long *out) {
    __shared__ uint32_t taddr;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = taddr + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128 % 512);
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c0 = 0; c0 < 4; c0 += kIn) {
            uint32_t v[kIn][32];
#pragma unroll
            for (int k = 0; k < kIn; ++k) {
                if (kPack) LD16P(v[k], base + (uint32_t)((c0 + k) * 32));
                else LD32(v[k], base + (uint32_t)((c0 + k) * 32));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < kIn; ++k) acc += v[k][k + 1];
        }
    }
    long long t1 = clock64();
    if (acc == 0x12345u) out[1000] = acc;
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr));
}

extern "C" int run_bw(int inflight, int pack, int threads, int iters, long long *out, void *st) {
    auto s = (cudaStream_t)st;
    if (pack) {
        if (inflight == 1) bw<1, true><<<148, threads, 0, s>>>(iters, out);
        else if (inflight == 2) bw<2, true><<<148, threads, 0, s>>>(iters, out);
        else bw<4, true><<<148, threads, 0, s>>>(iters, out);
    } else {
        if (inflight == 1) bw<1, false><<<148, threads, 0, s>>>(iters, out);
        else if (inflight == 2) bw<2, false><<<148, threads, 0, s>>>(iters, out);
        else bw<4, false><<<148, threads, 0, s>>>(iters, out);
    }
    return (int)cudaGetLastError();
}
