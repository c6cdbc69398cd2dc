// tri_common.cuh -- device/host primitives of the block-space map (sm_100a).
//
// "P:a-b" = PAPER.md lines.  The map lambda(omega) of Eq. 4 is
// evaluated from an fp32 MUFU reciprocal-sqrt estimate of sqrt(8 omega + 1)
// (the lambda_R idea of P:363-370) followed by ONE exact uint64 correction
// step each way against the row-boundary property Eq. 3, which
// replaces the paper's epsilon = 1e-4 patch.  The
// estimate is within +-1 row for every omega < 2^40 (verified exhaustively on
// the GPU by tri_map_eval), so lambda is exact on that range.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/tri.h"

#define TRI_HD __host__ __device__ __forceinline__

namespace tri {

TRI_HD uint64_t T2(uint64_t r) { return r * (r + 1) / 2; }
TRI_HD uint64_t T3(uint64_t r) { return r * (r + 1) * (r + 2) / 6; }

// Bare MUFU.RSQ: rsqrtf() adds a denormal-input rescale (FSETP + 2 FMUL + FSEL)
// around it; for normal inputs the MUFU result is the same.
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// fp32 estimate of sqrt(x): MUFU.RSQ on the device, libm on the host.  x = 8 w + 1
// >= 1 is never denormal.
TRI_HD float sqrt_est(float x) {
#ifdef __CUDA_ARCH__
    return x * rsqrt_ftz(x);   // MUFU.RSQ + FMUL (lambda_R form)
#else
    return sqrtf(x);
#endif
}

// lambda(omega) -> (bi, bj), Eq. 4 with the Eq. 3 integer correction.
TRI_HD void lambda_map(uint64_t w, uint32_t &bi, uint32_t &bj) {
    const float x = (float)(8ull * w + 1ull);
    const float s = sqrt_est(x);
    float e = (s - 1.0f) * 0.5f;
    e = e > 0.0f ? e : 0.0f;
    uint32_t i = (uint32_t)e;
    uint64_t t = T2(i);
    if (t > w) { t -= i; --i; }                      // T(i-1) = T(i) - i
    else if (t + i + 1 <= w) { t += i + 1; ++i; }    // T(i+1) = T(i) + i + 1
    bi = i;
    bj = (uint32_t)(w - t);
}

// Eq. 5, the map onto the STRICT lower triangle (no diagonal).  As
// printed its j-term gives (1, -1) at omega = 0; reading Q2 takes
// j = omega - i(i-1)/2 with i = floor(sqrt(1/4 + 2 omega) + 1/2), which equals
// (lambda(omega).i + 1, lambda(omega).j) -- computed that way, so it inherits
// lambda's integer correction and exactness.
TRI_HD void lambda_nodiag(uint64_t w, uint32_t &bi, uint32_t &bj) {
    uint32_t i, j;
    lambda_map(w, i, j);
    bi = i + 1;
    bj = j;
}

// The paper's three square-root variants of Eq. 4 (section 4.1),
// WITHOUT the integer correction -- exact only inside their validity range.
// Operations are explicit round-to-nearest intrinsics (no FMA contraction) so
// lambda_X and lambda_N are bit-reproducible on the CPU; lambda_R uses the
// hardware MUFU.RSQ approximation and is not.
//   lambda_X: i = floor(sqrtf(1/4 + 2 w) - 1/2)
//   lambda_N: sqrt by x * (0x5f3759df seed + 3 Newton steps) + eps
//   lambda_R: sqrt by x * rsqrtf(x) + eps
// eps = 1e-4.  Variant ids: TRI_SQRT_X / _N / _R (include/tri.h).

TRI_HD float sqrt_variant(float x, int variant) {
#ifdef __CUDA_ARCH__
    if (variant == TRI_SQRT_X) return __fsqrt_rn(x);
    if (variant == TRI_SQRT_R) return __fadd_rn(__fmul_rn(x, rsqrtf(x)), 1e-4f);
    // lambda_N: Carmack / Lomont reciprocal square root, three Newton steps in
    // the cited code's order y * (1.5 - (x2 * y) * y)
    const float xh = __fmul_rn(0.5f, x);
    float y = __int_as_float(0x5f3759df - (__float_as_int(x) >> 1));
#pragma unroll
    for (int it = 0; it < 3; ++it) y = __fmul_rn(y, __fsub_rn(1.5f, __fmul_rn(__fmul_rn(xh, y), y)));
    return __fadd_rn(__fmul_rn(x, y), 1e-4f);
#else
    (void)variant;
    return sqrtf(x);
#endif
}

// lambda with a sqrt variant, no correction: returns false if i would be negative.
TRI_HD void lambda_variant(uint64_t w, int variant, uint32_t &bi, uint32_t &bj) {
#ifdef __CUDA_ARCH__
    const float x = __fadd_rn(0.25f, __fmul_rn(2.0f, __ull2float_rn(w)));
    const float s = __fsub_rn(sqrt_variant(x, variant), 0.5f);
#else
    const float x = 0.25f + 2.0f * (float)w;
    const float s = sqrt_variant(x, variant) - 0.5f;
#endif
    const float f = floorf(s);
    const uint32_t i = f > 0.0f ? (uint32_t)f : 0u;
    bi = i;
    bj = (uint32_t)(w - T2(i));     // wraps when i is wrong: the self-check compares with exact lambda
}

// RB, the rectangular-box comparator map (Jung et al.; reading Q19:
// the printed "j = n - i - 1" is not a bijection, this fold is).  The lower
// triangle with diagonal is folded into an H x W thread rectangle,
// h = floor(n/2), H = n - h, W = 2h + 1 (W H = n(n+1)/2 exactly): rectangle row
// y holds triangle row a = h + y (x <= a -> (a, x)) followed by row b = h-1-y
// (x > a -> (b, x - a - 1)).  Thread-space, O(1) waste beyond block rounding.
TRI_HD bool rb_map(int64_t x, int64_t y, int64_t n, int64_t &i, int64_t &j) {
    const int64_t h = n / 2, H = n - h, W = 2 * h + 1;
    if (x >= W || y >= H) return false;
    const int64_t a = h + y;
    if (x <= a) { i = a; j = x; }
    else { i = h - 1 - y; j = x - a - 1; }
    return true;
}

// Tetrahedral map: k = largest layer with T3(k) <= omega from an
// fp32 cube-root estimate of (6 omega) (device: MUFU lg2/ex2, host: cbrtf) (the real root y = x + 1 of
// y^3 - y = 6 omega, reading Q13) plus one integer correction
// step each way; then (i, j) = lambda(omega - T3(k)).
// Device cube root as 2^(log2(x)/3) with the MUFU LG2 / EX2 approximations (relative
// error ~2^-21, far inside the +-1 row the integer correction absorbs; x = 0 gives
// 2^-inf = 0).  cbrtf() spends ~30 instructions on an exactly rounded result the
// correction does not need.
__device__ __forceinline__ float cbrt_est(float x) {
    float l, y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(l * (1.0f / 3.0f)));
    return y;
}

TRI_HD void tet_map(uint64_t w, uint32_t &i, uint32_t &j, uint32_t &k) {
#ifdef __CUDA_ARCH__
    const float c = cbrt_est((float)(6ull * w));
#else
    const float c = cbrtf((float)(6ull * w));
#endif
    float e = c - 1.0f;
    e = e > 0.0f ? e : 0.0f;
    uint32_t kk = (uint32_t)e;
    uint64_t t = T3(kk);
    if (t > w) { --kk; t = T3(kk); }
    else if (T3(kk + 1) <= w) { ++kk; t = T3(kk); }
    k = kk;
    lambda_map(w - t, i, j);
}

// Persistent lambda-walk: CTA c of the grid owns the contiguous
// omega chunk [begin + c*q + min(c, r), ...) of the balanced split of
// [begin, end) (q = nb / grid, r = nb % grid), evaluates lambda ONCE at the
// chunk start and then steps with the Eq. 1 successor rule (j + 1, wrapping to
// (i + 1, 0) past the diagonal).  Measured on B200: it wins where CTA launch is
// the cost (dummy kernel, n = 65536: 3.05 vs 6.25 ms) and loses on the
// HBM-write-bound kernels, whose packed rows end in the diagonal tile and
// resume in tile (i, 0) -- bi tiles earlier in omega, so in another CTA at
// another time -- leaving partial 32-B sectors to be read back from DRAM.
struct TileWalk {
    uint64_t w, end;
    uint32_t bi, bj;
    __device__ __forceinline__ TileWalk(uint64_t begin, uint64_t stop) {
        const uint64_t nb = stop - begin, g = gridDim.x, c = blockIdx.x;
        const uint64_t q = nb / g, r = nb % g;
        w = begin + c * q + (c < r ? c : r);
        end = w + q + (c < r ? 1 : 0);
        bi = bj = 0;
        if (w < end) lambda_map(w, bi, bj);
    }
    __device__ __forceinline__ bool more() const { return w < end; }
    __device__ __forceinline__ void next() {
        ++w;
        if (++bj > bi) { ++bi; bj = 0; }
    }
};

// Persistent CTAs with hardware work-stealing (sm_100 cluster launch control).
// The grid is the full lambda grid; a running CTA, after finishing a tile,
// cancels the next not-yet-launched CTA (clusterlaunchcontrol.try_cancel) and
// processes that CTA's tile instead, so tiles keep the hardware's omega-order
// dispatch (neighbouring tiles in flight together) while the CTA prologue,
// shared-memory setup and L1 contents persist.  One 16-B response + one
// mbarrier per CTA, in shared memory.
struct ClcSched {
    uint4 handle;
    unsigned long long mbar;
    __device__ __forceinline__ uint32_t hs() const { return (uint32_t)__cvta_generic_to_shared(&handle); }
    __device__ __forceinline__ uint32_t mb() const { return (uint32_t)__cvta_generic_to_shared(&mbar); }
    // one thread, before the first request; a __syncthreads() must follow
    __device__ __forceinline__ void init() {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb()));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // one thread: ask for the next CTA (asynchronous; the response lands in handle)
    __device__ __forceinline__ void request() {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(mb()) : "memory");
        asm volatile(
            "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];" ::"r"(
                hs()),
            "r"(mb())
            : "memory");
    }
    // every thread: wait for the response; returns false when no CTA was left.
    // The caller must __syncthreads() before the next request() reuses handle.
    __device__ __forceinline__ bool receive(uint32_t &phase, uint32_t &bx, uint32_t &by) {
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p;\n"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                "selp.b32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(mb()), "r"(phase)
                : "memory");
        phase ^= 1u;
        uint32_t ok, x, y, z;
        asm volatile(
            "{ .reg .b128 h; .reg .pred p;\n"
            "ld.shared.b128 h, [%4];\n"
            "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, h;\n"
            "selp.b32 %0, 1, 0, p;\n"
            "clusterlaunchcontrol.query_cancel.get_first_ctaid.v4.b32.b128 {%1, %2, %3, _}, h; }"
            : "=r"(ok), "=r"(x), "=r"(y), "=r"(z)
            : "r"(hs())
            : "memory");
        // order this generic-proxy read before the next request's async-proxy write
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bx = x;
        by = y;
        return ok != 0;
    }
};

}  // namespace tri

// ------------------------------------------------------------------ device stores
__device__ __forceinline__ void st_cs_v4(float *p, float a, float b, float c, float d) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d) : "memory");
}
__device__ __forceinline__ void st_cs_v4u(void *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c),
                 "r"(d) : "memory");
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));   // MUFU.SQRT, no denormal fix-up
    return y;
}

// ------------------------------------------------------------------ internal launch API
namespace tri {

// Per-call launch bookkeeping (thread-local in abi.cu).
void note_launches(int k);
void reset_launches();
int sm_count();                       // SMs of the current device (cached)
inline tri_status cuda_status() {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TRI_OK : TRI_ECUDA;
}

// Grid helper for lambda launches: nb tiles as (gx, gy) with gx*gy >= nb.
inline dim3 tile_grid(uint64_t nb) {
    const uint64_t gx_max = 1ull << 30;
    uint64_t gx = nb < gx_max ? nb : gx_max;
    if (gx == 0) gx = 1;
    uint64_t gy = (nb + gx - 1) / gx;
    return dim3((unsigned)gx, (unsigned)(gy ? gy : 1), 1);
}

size_t ca_run_ws_bytes(const tri_map_t &m);
tri_status launch_ca_run(const tri_map_t &m, int strategy, int64_t steps, const uint8_t *in, uint8_t *out,
                         void *ws, cudaStream_t st);

// Shared argument validation of tri_edm / tri_edm_host (abi.cu): true = EINVAL.
bool edm_args_bad(const tri_map_t *map, int32_t strategy, int32_t dim, int64_t ld, size_t pts_bytes,
                  size_t out_bytes);

// Kernel launchers (one per .cu file); args validated by abi.cu.
tri_status launch_map_eval(uint64_t w0, uint64_t count, uint32_t *d_ij, unsigned long long *d_fail,
                           cudaStream_t st);
tri_status launch_tet_map_eval(uint64_t w0, uint64_t count, uint32_t *d_ijk,
                               unsigned long long *d_fail, cudaStream_t st);
tri_status launch_tet_lut_build(uint32_t kmax, int shift, void *d_lut, cudaStream_t st);
tri_status launch_tet_map_eval_lut(uint64_t w0, uint64_t count, uint32_t kmax, int shift, const void *d_lut,
                                   uint32_t *d_ijk, unsigned long long *d_fail, cudaStream_t st);
tri_status launch_variant_scan(int variant, uint64_t w0, uint64_t count, unsigned long long *d_fail,
                               unsigned long long *d_first, cudaStream_t st);
tri_status launch_variant_rows(int variant, uint64_t w0, uint64_t count, uint32_t *d_rows, cudaStream_t st);
tri_status launch_dummy_rb(const tri_map_t &m, int mode, void *d_out, cudaStream_t st);
tri_status launch_collide_tc(const tri_map_t &m, int strategy, const float *sph, unsigned long long *count,
                             void *ws, cudaStream_t st);
size_t collide_tc_ws_bytes(const tri_map_t &m);
tri_status launch_tc_tf32_probe(const float *x, const float *y, float *d, cudaStream_t st);
tri_status launch_tc_f16_probe(const void *x, const void *y, void *d, cudaStream_t st);
tri_status launch_collide1d(const tri_map_t &m, int strategy, const float *iv, unsigned long long *count,
                            cudaStream_t st);
tri_status launch_ca_steps(const tri_map_t &m, int strategy, int k, const uint8_t *in, uint8_t *out,
                           const uint8_t *above, const uint8_t *below, uint8_t *peer_above, uint8_t *peer_below,
                           cudaStream_t st);
tri_status launch_edm_rb(const tri_map_t &m, const float *pts, int dim, int64_t ld, float *out, cudaStream_t st);
tri_status launch_dummy(const tri_map_t &m, int strategy, int mode, void *d_out, cudaStream_t st);
tri_status launch_edm(const tri_map_t &m, int strategy, const float *pts, int dim, int64_t ld,
                      float *out, cudaStream_t st);
tri_status launch_collide(const tri_map_t &m, int strategy, const float *sph,
                          unsigned long long *count, cudaStream_t st);
tri_status launch_ca(const tri_map_t &m, int strategy, const uint8_t *in, uint8_t *out,
                     const uint8_t *above, const uint8_t *below, cudaStream_t st);
tri_status launch_triplet(const tet_map_t &m, int strategy, const float *pts, double nu,
                          double *energy, cudaStream_t st);

}  // namespace tri
