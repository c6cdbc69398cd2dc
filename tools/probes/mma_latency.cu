// Microbenchmark (tools only, not product): latency and throughput of one-thread-issued
// tcgen05.mma.kind::tf32 128 x N x 8 with no-swizzle K-major operands, commit -> mbarrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o _ab/libmma.so tools/probes/mma_latency.cu
// run_probe(mode, n_cols, iters, out) with one CTA per SM; out[cta] = cycles per iteration.
//   mode 0: issue 1 MMA, commit, try_wait          (round-trip latency)
//   mode 1: issue 1 MMA, commit, test_wait spin    (round-trip latency, no suspend)
//   mode 2: issue 4 MMAs into 4 accumulators, one commit each, wait all   (4 in flight)
//   mode 3: issue 16 MMAs (4 accumulators x 4), one commit, wait          (pure issue stream)
//   mode 4: mode 0 with the accumulator also drained by tcgen05.ld by 4 warps each time
//   mode 5: no MMA: each warp re-reads its lane quarter of 128 columns (4 x .x32 in flight, one wait)
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);
    d |= (uint64_t)(128 >> 4) << 16;
    d |= (uint64_t)(256 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

template <int N>
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc) {
    constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                 "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t mb) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb) : "memory");
}
__device__ __forceinline__ void wait_try(uint32_t mb, uint32_t par) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}\n"
                     : "=r"(done) : "r"(mb), "r"(par) : "memory");
}
__device__ __forceinline__ void wait_test(uint32_t mb, uint32_t par) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}\n"
                     : "=r"(done) : "r"(mb), "r"(par) : "memory");
}

template <int N>
__global__ void __launch_bounds__(512, 1) probe(int mode, int iters, long long *out) {
    __shared__ __align__(1024) uint32_t sa[128 * 8], sb[256 * 8];
    __shared__ __align__(8) unsigned long long bar[5];
    __shared__ uint32_t taddr;
    const int t = threadIdx.x, warp = t >> 5;
    for (int k = t; k < 128 * 8; k += blockDim.x) sa[k] = 0x3f800000u;
    for (int k = t; k < 256 * 8; k += blockDim.x) sb[k] = 0x3f800000u;
    if (t == 0) {
        for (int k = 0; k < 5; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[k])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = taddr;
    const uint64_t da = desc((uint32_t)__cvta_generic_to_shared(sa)), db = desc((uint32_t)__cvta_generic_to_shared(sb));
    uint32_t mb[5];
    for (int k = 0; k < 5; ++k) mb[k] = (uint32_t)__cvta_generic_to_shared(&bar[k]);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode == 0 || mode == 1 || mode == 4) {
            if (t == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;");
                mma<N>(tmem, da, db, 0);
                commit(mb[0]);
            }
            if (mode == 1) wait_test(mb[0], ph); else wait_try(mb[0], ph);
            ph ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (mode == 4) {
                uint32_t v[32];
                for (int cg = 0; cg < N / 32; ++cg) {
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + cg * 32));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (v[7] == 12345u) out[1000] = v[3];
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncthreads();
        } else if (mode == 5) {
            uint32_t v[4][32];
#pragma unroll
            for (int cg = 0; cg < 4; ++cg)
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                             : "=r"(v[cg][0]), "=r"(v[cg][1]), "=r"(v[cg][2]), "=r"(v[cg][3]), "=r"(v[cg][4]), "=r"(v[cg][5]), "=r"(v[cg][6]), "=r"(v[cg][7]), "=r"(v[cg][8]), "=r"(v[cg][9]), "=r"(v[cg][10]), "=r"(v[cg][11]), "=r"(v[cg][12]), "=r"(v[cg][13]), "=r"(v[cg][14]), "=r"(v[cg][15]), "=r"(v[cg][16]), "=r"(v[cg][17]), "=r"(v[cg][18]), "=r"(v[cg][19]), "=r"(v[cg][20]), "=r"(v[cg][21]), "=r"(v[cg][22]), "=r"(v[cg][23]), "=r"(v[cg][24]), "=r"(v[cg][25]), "=r"(v[cg][26]), "=r"(v[cg][27]), "=r"(v[cg][28]), "=r"(v[cg][29]), "=r"(v[cg][30]), "=r"(v[cg][31])
                             : "r"(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(((warp >> 2) * 128 + cg * 32) & 511)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            uint32_t x = 0;
#pragma unroll
            for (int cg = 0; cg < 4; ++cg)
#pragma unroll
                for (int e = 0; e < 32; ++e) x ^= v[cg][e];
            if (x == 0x12345u) out[1000 + t] = x;
        } else if (mode == 2) {
            if (t == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;");
                for (int k = 0; k < 4; ++k) { mma<N>(tmem + k * 128, da, db, 0); commit(mb[1 + k]); }
            }
            for (int k = 0; k < 4; ++k) wait_try(mb[1 + k], ph);
            ph ^= 1;
            __syncthreads();
        } else {
            if (t == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;");
                for (int k = 0; k < 16; ++k) mma<N>(tmem + (k & 3) * 128, da, db, k >= 4);
                commit(mb[0]);
            }
            wait_try(mb[0], ph);
            ph ^= 1;
            __syncthreads();
        }
    }
    long long t1 = clock64();
    if (t == 0) out[blockIdx.x] = (t1 - t0) / iters;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

extern "C" int run_probe(int mode, int ncols, int iters, int grid, long long *out, void *st, int threads) {
    if (ncols == 128) probe<128><<<grid, threads, 0, (cudaStream_t)st>>>(mode, iters, out);
    else if (ncols == 64) probe<64><<<grid, threads, 0, (cudaStream_t)st>>>(mode, iters, out);
    else probe<256><<<grid, threads, 0, (cudaStream_t)st>>>(mode, iters, out);
    return (int)cudaGetLastError();
}
