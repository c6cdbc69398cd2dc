// Probe (tools only): tcgen05.mma.kind::f16 (fp16 A/B, K = 16) into an F16 or F32
// accumulator, M = 128, N = 128.  Reports the raw TMEM words of columns [0, 256) so the
// host can see how a 16-bit accumulator is laid out, and the values for a precision check.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o _ab/libf16acc.so tools/probes/f16acc.cu
// run_f16(a, b, out, dfmt, stream): a, b = 128 x 16 fp16 row-major; out = 128 x 256 u32.
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);
    d |= (uint64_t)(128 >> 4) << 16;
    d |= (uint64_t)(256 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__global__ void __launch_bounds__(128, 1) f16probe(const uint16_t *a, const uint16_t *b, uint32_t *out, int dfmt) {
    __shared__ __align__(1024) uint16_t sa[128 * 16], sb[128 * 16];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ uint32_t taddr;
    const int t = threadIdx.x, warp = t >> 5;
    // canonical K-major no-swizzle: row r, element k (16-bit) -> group r/8 (256 B), K half k/8 (+128 B), row r%8 (+16 B)
    for (int k = 0; k < 16; ++k) {
        const int idx = (t >> 3) * 128 + (k >> 3) * 64 + (t & 7) * 8 + (k & 7);
        sa[idx] = a[t * 16 + k];
        sb[idx] = b[t * 16 + k];
    }
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar);
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = taddr;
    // sentinel in every column
    {
        uint32_t s = 0xDEADBEEFu;
        for (int c = 0; c < 256; ++c)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + c), "r"(s));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (t == 0) {
        const uint32_t idesc = ((uint32_t)dfmt << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t da = desc((uint32_t)__cvta_generic_to_shared(sa)), db = desc((uint32_t)__cvta_generic_to_shared(sb));
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb) : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.b32 %0, 1, 0, p;\n\t}\n"
                     : "=r"(done) : "r"(mb) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c = 0; c < 256; ++c) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[t * 256 + c] = v;
    }
    if (dfmt == 0) {   // packed load of columns 0..31 into 16 registers -> out columns 128..143
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int c = 0; c < 16; ++c) out[t * 256 + 128 + c] = v[c];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

extern "C" int run_f16(const void *a, const void *b, void *out, int dfmt, void *st) {
    f16probe<<<1, 128, 0, (cudaStream_t)st>>>((const uint16_t *)a, (const uint16_t *)b, (uint32_t *)out, dfmt);
    return (int)cudaGetLastError();
}
