# Probe patch (not product code): clock64 phase trace of collide_tc_kernel on SM 0.
# Usage: bash tools/ab_variant.sh trace tools/probes/tc_trace_patch.py; python tools/probes/tc_trace.py _ab/libtri_trace.so
s=open('csrc/collide_tc.cu').read()
# global trace buffer
s=s.replace('''template <int kRho, bool kBB>
__global__ void __launch_bounds__(kTileThreads, kCtasPerSm) collide_tc_kernel(TcArgs a) {''','''__device__ unsigned long long g_trace[1 << 20];
__device__ unsigned int g_trace_n;
__shared__ unsigned long long g_ts[64][6];
__device__ __forceinline__ void tr(int ev, int idx) { g_ts[idx & 63][ev] = clock64(); }
__device__ __forceinline__ void tr_flush(int nblk) {
    unsigned smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (smid != 0) return;
    const unsigned k = atomicAdd(&g_trace_n, (unsigned)(nblk * 6));
    for (int i = 0; i < nblk; ++i)
        for (int e = 0; e < 6; ++e)
            if (k + i * 6 + e < (1u << 20))
                g_trace[k + i * 6 + e] = ((unsigned long long)g_ts[i][e] << 24) | ((unsigned long long)(blockIdx.x & 0xffff) << 8) | ((unsigned)e << 5) | (i & 31);
}
template <int kRho, bool kBB>
__global__ void __launch_bounds__(kTileThreads, kCtasPerSm) collide_tc_kernel(TcArgs a) {''')
s=s.replace('''        mbar_wait(mb_mma + 8 * acc, (uint32_t)(kAccs == 1 ? idx : idx >> 1) & 1u, a.count);
        asm volatile("tcgen05.fence::after_thread_sync;");''','''        if (t == 0) tr(0, idx);
        mbar_wait(mb_mma + 8 * acc, (uint32_t)(kAccs == 1 ? idx : idx >> 1) & 1u, a.count);
        if (t == 0) tr(1, idx);
        asm volatile("tcgen05.fence::after_thread_sync;");''')
s=s.replace('''        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // the accumulator is in registers''','''        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (t == 0) tr(2, idx);
        // the accumulator is in registers''')
s=s.replace('''        if (t == 0 && idx + kAccs < nblk) issue(idx + kAccs);
        uint32_t o[NG], any = 0;''','''        if (t == 0) tr(3, idx);
        if (t == 0 && idx + kAccs < nblk) issue(idx + kAccs);
        if (t == 0) tr(4, idx);
        uint32_t o[NG], any = 0;''')
s=s.replace('''        if (any & 0x80008000u) {                           // rare''','''        if (t == 0) { asm volatile("" :: "r"(any)); tr(5, idx); }
        if (any & 0x80008000u) {                           // rare''')
s=s.replace('''    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc''', '''    if (t == 0) tr_flush(nblk);
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc''', 1)
s+='''
extern "C" int tri_tc_trace(void *host, unsigned *n) {
    cudaMemcpyFromSymbol(n, g_trace_n, sizeof(unsigned));
    unsigned m = *n < (1u << 20) ? *n : (1u << 20);
    cudaMemcpyFromSymbol(host, g_trace, m * 8ull);
    unsigned z = 0; cudaMemcpyToSymbol(g_trace_n, &z, 4);
    return (int)cudaGetLastError();
}
'''
open('csrc/collide_tc.cu','w').write(s)
