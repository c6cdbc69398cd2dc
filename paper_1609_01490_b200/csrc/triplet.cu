// triplet.cu -- triplet-interaction n-body energy on the tetrahedral map
// (interaction = Axilrod-Teller-Muto,
// DESIGN.md reading Q15).
//
// Tile (i, j, k), j <= i <= k, from the tetrahedral lambda (P:617-654 with the
// integer correction) or a BB-3D m^3 grid whose tiles outside j <= i <= k exit
// (the 3-D analogue of P:411-418).  Particle blocks: p in layer block k, q in
// block i, s in block j; strict p > q > s is filtered per triplet on the
// tiles where two block indices coincide.
// Thread (tz, ty) owns the pair (p, q) = (k rho + tz, i rho + ty) -- so
// a = |x_p - x_q|^2 lives in a register -- and loops over the rho particles s
// of block j, reading b = |x_q - x_s|^2 and c = |x_s - x_p|^2 from two rho x rho
// pair-distance tables built once per tile in shared memory (read as float4).
// Per triplet (fp32): abc, P = (b+c-a)(a-(b-c))(a+(b-c)), r = rsqrt(abc),
// E = r^3 (1 + 0.375 P r^2).  E/3 is credited to p, q and s:
//   * p and q: the thread's running sum (fp64 across tiles, flushed when the
//     (k, i) pair changes -- consecutive tetrahedral tiles share it);
//   * s: a per-thread es[rho] register array, reduce-scattered across the warp
//     with butterfly shuffles, summed over warps in shared memory;
// all flushed with fp64 RED.ADD into d_energy.
#include "tri_common.cuh"

namespace {

struct TripArgs {
    const float4 *pts;
    int64_t n;
    double nu_third;
    double *energy;
    uint64_t omega_begin, omega_end;
    uint32_t m;
};

template <int RHO>
struct TripSmem {
    float4 P[RHO], Q[RHO], S[RHO];
    float Dqs[RHO][RHO];   // [q][s]
    float Dps[RHO][RHO];   // [p][s]
    float red[(RHO * RHO) / 32][RHO];
    double acc[RHO][RHO];  // [p][q] flush buffer
};

__device__ __forceinline__ float d2(const float4 a, const float4 b) {
    const float dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
    return fmaf(dz, dz, fmaf(dy, dy, dx * dx));
}

// ATM energy (without nu) from squared side lengths.
__device__ __forceinline__ float atm(float a, float b, float c) {
    const float abc = a * b * c;
    const float bc = b + c, dbc = b - c;
    const float P = (bc - a) * (a - dbc) * (a + dbc);
    const float r = tri::rsqrt_ftz(abc);         // abc < 2^-126 overflows E (r^9) anyway
    const float r2 = r * r;
    const float r3 = r2 * r;
    return fmaf(0.375f * P * r2, r3, r3);
}

// Reduce-scatter of V per-lane values across the warp: afterwards lane l holds
// in v[0] the warp total of index idx(l); returns idx(l).  Butterfly halving.
template <int V>
__device__ __forceinline__ int reduce_scatter(float (&v)[V], int lane) {
    int idx = 0;
    int half = V / 2;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        if (half >= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int h = 0; h < V / 2; ++h) {
                if (h < half) {
                    const float send = up ? v[h] : v[h + half];
                    const float keep = up ? v[h + half] : v[h];
                    v[h] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            idx += up ? half : 0;
            half >>= 1;
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        }
    }
    return idx;
}

template <int RHO>
__device__ __forceinline__ void flush_pq(const TripArgs &a, TripSmem<RHO> &sm, double acc, uint32_t kb,
                                         uint32_t ib) {
    const int t = threadIdx.x, ty = t % RHO, tz = t / RHO;
    sm.acc[tz][ty] = acc;
    __syncthreads();
    if (t < RHO) {
        double s = 0;
#pragma unroll 4
        for (int q = 0; q < RHO; ++q) s += sm.acc[t][q];
        const int64_t p = (int64_t)kb * RHO + t;
        if (s != 0.0 && p < a.n) atomicAdd(a.energy + p, s * a.nu_third);
    } else if (t < 2 * RHO) {
        const int qq = t - RHO;
        double s = 0;
#pragma unroll 4
        for (int p = 0; p < RHO; ++p) s += sm.acc[p][qq];
        const int64_t q = (int64_t)ib * RHO + qq;
        if (s != 0.0 && q < a.n) atomicAdd(a.energy + q, s * a.nu_third);
    }
    __syncthreads();
}

// One tile; returns this thread's fp32 sum over s of E(p, q, s).  Credits s.
template <int RHO>
__device__ __forceinline__ float triplet_tile(const TripArgs &a, TripSmem<RHO> &sm, uint32_t kb, uint32_t ib,
                                              uint32_t jb) {
    constexpr int NT = RHO * RHO;
    const int t = threadIdx.x, ty = t % RHO, tz = t / RHO, lane = t & 31, warp = t >> 5;
    if (t < 3 * RHO) {
        const int g = t / RHO, x = t % RHO;
        const uint32_t blk = g == 0 ? kb : (g == 1 ? ib : jb);
        const int64_t idx = (int64_t)blk * RHO + x;
        const float4 v = idx < a.n ? __ldg(a.pts + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
        (g == 0 ? sm.P : (g == 1 ? sm.Q : sm.S))[x] = v;
    }
    __syncthreads();
    // tables: thread (row = tz, col = ty)
    sm.Dqs[tz][ty] = d2(sm.Q[tz], sm.S[ty]);
    sm.Dps[tz][ty] = d2(sm.P[tz], sm.S[ty]);
    const float A = d2(sm.P[tz], sm.Q[ty]);
    __syncthreads();
    const int64_t p = (int64_t)kb * RHO + tz, q = (int64_t)ib * RHO + ty;
    const bool pq_ok = p < a.n && q < a.n && (kb != ib || tz > ty);
    const int64_t s_lim = a.n - (int64_t)jb * RHO;          // s_local < s_lim
    const int s_max = (ib == jb) ? ty : RHO;                 // s_local < s_max (strict q > s)
    float es[RHO];
    float acc = 0.f;
#pragma unroll
    for (int s4 = 0; s4 < RHO / 4; ++s4) {
        const float4 b4 = *reinterpret_cast<const float4 *>(&sm.Dqs[ty][4 * s4]);
        const float4 c4 = *reinterpret_cast<const float4 *>(&sm.Dps[tz][4 * s4]);
        const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
        const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int sl = 4 * s4 + u;
            const bool ok = pq_ok && sl < s_max && sl < s_lim;
            const float E = ok ? atm(A, bb[u], cc[u]) : 0.f;
            acc += E;
            es[sl] = E;
        }
    }
    // credit s: warp reduce-scatter, then across warps
    const int idx = reduce_scatter<RHO>(es, lane);
    constexpr int KEEP = 32 / RHO;   // lanes holding the same index after the butterfly
    if ((lane % KEEP) == 0 || KEEP <= 1) sm.red[warp][idx] = es[0];
    __syncthreads();
    if (t < RHO) {
        double s = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) s += (double)sm.red[w][t];
        const int64_t si = (int64_t)jb * RHO + t;
        if (s != 0.0 && si < a.n) atomicAdd(a.energy + si, s * a.nu_third);
    }
    return acc;
}

template <int RHO, int STRAT>
__global__ void __launch_bounds__(RHO *RHO) triplet_kernel(TripArgs a) {
    __shared__ __align__(16) TripSmem<RHO> sm;
    if (STRAT == TRI_BB) {
        const uint32_t jb = blockIdx.x, ib = blockIdx.y, kb = blockIdx.z;
        if (jb > ib || ib > kb) return;                         // outside the tetrahedron
        const float acc = triplet_tile<RHO>(a, sm, kb, ib, jb);
        flush_pq<RHO>(a, sm, (double)acc, kb, ib);
    } else if (STRAT == TRI_LAMBDA) {
        const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (w >= a.omega_end) return;
        uint32_t ib, jb, kb;
        tri::tet_map(w, ib, jb, kb);
        const float acc = triplet_tile<RHO>(a, sm, kb, ib, jb);
        flush_pq<RHO>(a, sm, (double)acc, kb, ib);
    } else {
        // contiguous omega chunk per CTA: consecutive tiles share (k, i)
        const uint64_t nb = a.omega_end - a.omega_begin;
        const uint64_t per = (nb + gridDim.x - 1) / gridDim.x;
        const uint64_t w0 = a.omega_begin + per * blockIdx.x;
        uint64_t w1 = w0 + per;
        if (w1 > a.omega_end) w1 = a.omega_end;
        if (w0 >= w1) return;
        uint32_t ib, jb, kb;
        tri::tet_map(w0, ib, jb, kb);
        double acc = 0;
#pragma unroll 1
        for (uint64_t w = w0; w < w1; ++w) {
            acc += (double)triplet_tile<RHO>(a, sm, kb, ib, jb);
            // successor in layer-major Eq. 1 order
            uint32_t nj = jb + 1, ni = ib, nk = kb;
            if (nj > ni) { nj = 0; ++ni; }
            if (ni > nk) { ni = 0; ++nk; }
            if (ni != ib || nk != kb || w + 1 == w1) {
                flush_pq<RHO>(a, sm, acc, kb, ib);
                acc = 0;
            } else {
                __syncthreads();   // smem tables reused by the next tile
            }
            ib = ni; jb = nj; kb = nk;
        }
    }
}

template <int RHO>
tri_status launch_r(const tet_map_t &m, int strategy, TripArgs a, cudaStream_t st) {
    constexpr int NT = RHO * RHO;
    if (strategy == TRI_BB) {
        if (m.world > 1) return TRI_ENOTSUP;
        if (m.m > 65535) return TRI_ENOTSUP;
        const unsigned mm = (unsigned)m.m;
        triplet_kernel<RHO, TRI_BB><<<dim3(mm, mm, mm), NT, 0, st>>>(a);
    } else if (strategy == TRI_LAMBDA) {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        triplet_kernel<RHO, TRI_LAMBDA><<<tri::tile_grid(nb), NT, 0, st>>>(a);
    } else {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, triplet_kernel<RHO, TRI_LAMBDA_PERSIST>, NT, 0);
        uint64_t g = (uint64_t)tri::sm_count() * (uint64_t)(per_sm > 0 ? per_sm : 1);
        if (g > nb) g = nb;
        triplet_kernel<RHO, TRI_LAMBDA_PERSIST><<<(unsigned)g, NT, 0, st>>>(a);
    }
    tri::note_launches(1);
    return tri::cuda_status();
}

// ============================================================================
// rho = 32: one WARP per tetrahedral tile.  Lane l owns p = k*32 + l and walks
// all (q, s) of the tile (1024 triplets per lane), so
//   * e_p accumulates in the lane's register (fp64 across tiles with equal k),
//   * e_q is one warp all-reduce per q (lane q keeps it; fp64 across tiles with
//     equal (k, i)),
//   * e_s is a 32-value register vector reduce-scattered across the warp once
//     per tile (~0.12 shuffles per triplet).
// Two squared-distance tables per warp live in shared memory, padded so every
// access pattern is conflict-free: Dps[p][s] (stride 36, per-lane LDS.128) and
// Dqs[q][s] (stride 32, broadcast LDS.128); a = |x_p - x_q|^2 is recomputed per
// q (5 ops per 32 triplets -- cheaper than the 4 KB table it replaces, which
// bought occupancy: 5.52 -> 5.35 ms).  Two s values are processed per
// instruction with the packed sm_100 f32x2 ops; MUFU.RSQ stays scalar.
//   E = r^3 (1 + P' r^2), r = (abc)^-1/2, P' = 3/8 (b+c-a)(a-b+c)(a+b-c)
// (see atm2 for the operation order).
namespace t32 {

typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk(f2 v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
#define T32_OP2(name, op)                                                          \
    __device__ __forceinline__ f2 name(f2 a, f2 b) {                               \
        f2 r;                                                                      \
        asm(op " %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));                         \
        return r;                                                                  \
    }
T32_OP2(add2, "add.rn.f32x2")
T32_OP2(sub2, "sub.rn.f32x2")
T32_OP2(mul2, "mul.rn.f32x2")
#undef T32_OP2
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Two ATM energies (without nu) for the s-pair (b, c) at fixed a, 10 FP32 ops each:
//   P' = 3/8 P = (0.375 a - 0.375 (b + c)) * ((b - c)^2 - a^2)     (both factors negated)
//   E  = r^3 (1 + P' r^2),  r = rsqrt(a b c)      (0.375 a and -a^2 hoisted per q)
// Returns E as the product r3 * y so the caller can fuse it into its accumulators.
__device__ __forceinline__ void atm2(f2 aa, f2 na2, f2 a375, f2 nc375, f2 one, f2 b, f2 c, f2 &r3, f2 &y) {
    const f2 sg = add2(b, c), dl = sub2(b, c);
    const f2 u = fma2(nc375, sg, a375);                  // 0.375 (a - b - c)
    const f2 t = fma2(dl, dl, na2);                       // (b - c)^2 - a^2
    const f2 P = mul2(u, t);
    float x0, x1;
    upk(mul2(mul2(b, c), aa), x0, x1);
    // bare MUFU.RSQ (no denormal rescale): abc < 2^-126 would give E = r^9 > 2^567,
    // an fp32 overflow (inf) either way
    const f2 r = pk(tri::rsqrt_ftz(x0), tri::rsqrt_ftz(x1));
    const f2 r2 = mul2(r, r);
    y = fma2(P, r2, one);
    r3 = mul2(r2, r);
}

struct WarpSmem {
    float4 P[32], Q[32], S[32];
    float Dqs[32][32];
    float Dps[32][36];
};

__device__ __forceinline__ float d2f(const float4 a, const float4 b) {
    const float dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
    return fmaf(dz, dz, fmaf(dy, dy, dx * dx));
}

__device__ __forceinline__ float4 ldp(const TripArgs &a, int64_t idx) {
    return idx < a.n ? __ldg(a.pts + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
}

// Per-warp tile state carried across consecutive tiles.
struct Acc {
    double ep, eq;           // lane's p (block kb) and q (block ib) energies
    uint32_t kb, ib;
    bool live;
};

__device__ __forceinline__ void flush_pq(const TripArgs &a, Acc &acc, int lane) {
    if (!acc.live) return;
    const int64_t p = (int64_t)acc.kb * 32 + lane, q = (int64_t)acc.ib * 32 + lane;
    if (acc.ep != 0.0 && p < a.n) atomicAdd(a.energy + p, acc.ep * a.nu_third);
    if (acc.eq != 0.0 && q < a.n) atomicAdd(a.energy + q, acc.eq * a.nu_third);
    acc.ep = acc.eq = 0.0;
    acc.live = false;
}

template <bool MASKED>
__device__ __forceinline__ void tile(const TripArgs &a, WarpSmem &sm, uint32_t kb, uint32_t ib, uint32_t jb,
                                     bool new_pq, Acc &acc) {
    const int lane = threadIdx.x & 31;
    // stage points and tables (Dpq only when (k, i) changed)
    sm.S[lane] = ldp(a, (int64_t)jb * 32 + lane);
    if (new_pq) {
        sm.P[lane] = ldp(a, (int64_t)kb * 32 + lane);
        sm.Q[lane] = ldp(a, (int64_t)ib * 32 + lane);
    }
    __syncwarp();
    const float4 myS = sm.S[lane];
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
        sm.Dqs[r][lane] = d2f(sm.Q[r], myS);
        sm.Dps[r][lane] = d2f(sm.P[r], myS);
    }

    __syncwarp();
    const int64_t p = (int64_t)kb * 32 + lane;
    const float4 myP = sm.P[lane];
    const f2 nc375 = pk(-0.375f, -0.375f), one = pk(1.f, 1.f);
    f2 es[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) es[t] = 0ull;
    float accp = 0.f, myq = 0.f;
#pragma unroll 1
    for (int q = 0; q < 32; ++q) {
        const float av = d2f(myP, sm.Q[q]);                 // a = |x_p - x_q|^2, recomputed per q
        const f2 aa = pk(av, av), a375 = pk(0.375f * av, 0.375f * av), na2 = pk(-av * av, -av * av);
        f2 row = 0ull, row2 = 0ull;
        bool pq_ok = true;
        if (MASKED) pq_ok = p < a.n && (kb != ib || lane > q) && ((int64_t)ib * 32 + q < a.n);
#pragma unroll
        for (int s4 = 0; s4 < 8; ++s4) {
            const float4 b4 = *reinterpret_cast<const float4 *>(&sm.Dqs[q][4 * s4]);
            const float4 c4 = *reinterpret_cast<const float4 *>(&sm.Dps[lane][4 * s4]);
            f2 r01, y01, r23, y23;
            atm2(aa, na2, a375, nc375, one, pk(b4.x, b4.y), pk(c4.x, c4.y), r01, y01);
            atm2(aa, na2, a375, nc375, one, pk(b4.z, b4.w), pk(c4.z, c4.w), r23, y23);
            if (MASKED) {
                f2 e01 = mul2(r01, y01), e23 = mul2(r23, y23);
                float e0, e1, e2, e3;
                upk(e01, e0, e1);
                upk(e23, e2, e3);
                const int sb = 4 * s4;
                const int64_t sg = (int64_t)jb * 32 + sb;
                const bool sj = ib != jb;
                e0 = (pq_ok && sg + 0 < a.n && (sj || sb + 0 < q)) ? e0 : 0.f;
                e1 = (pq_ok && sg + 1 < a.n && (sj || sb + 1 < q)) ? e1 : 0.f;
                e2 = (pq_ok && sg + 2 < a.n && (sj || sb + 2 < q)) ? e2 : 0.f;
                e3 = (pq_ok && sg + 3 < a.n && (sj || sb + 3 < q)) ? e3 : 0.f;
                e01 = pk(e0, e1);
                e23 = pk(e2, e3);
                row = add2(row, e01);
                row2 = add2(row2, e23);
                es[2 * s4] = add2(es[2 * s4], e01);
                es[2 * s4 + 1] = add2(es[2 * s4 + 1], e23);
            } else {
                // E = r3 y fused into both accumulators
                row = fma2(r01, y01, row);
                row2 = fma2(r23, y23, row2);
                es[2 * s4] = fma2(r01, y01, es[2 * s4]);
                es[2 * s4 + 1] = fma2(r23, y23, es[2 * s4 + 1]);
            }
        }
        float r0, r1;
        upk(add2(row, row2), r0, r1);
        const float rs = r0 + r1;          // sum over s of E(p, q, s) for this lane's p
        accp += rs;
        float tq = rs;                     // sum over p (lanes) -> e_q
#pragma unroll
        for (int o = 16; o; o >>= 1) tq += __shfl_xor_sync(0xffffffffu, tq, o);
        myq = (lane == q) ? tq : myq;
    }
    acc.ep += (double)accp;
    acc.eq += (double)myq;
    acc.live = true;
    acc.kb = kb;
    acc.ib = ib;
    // e_s: reduce-scatter the 32 per-lane values over the warp (butterfly)
    float v[32];
#pragma unroll
    for (int t = 0; t < 16; ++t) upk(es[t], v[2 * t], v[2 * t + 1]);
    int idx = 0;
#pragma unroll
    for (int o = 16, half = 16; o >= 1; o >>= 1, half >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int h = 0; h < half; ++h) {
            const float send = up ? v[h] : v[h + half];
            const float keep = up ? v[h + half] : v[h];
            v[h] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
        idx += up ? half : 0;
    }
    const int64_t si = (int64_t)jb * 32 + idx;
    if (v[0] != 0.f && si < a.n) atomicAdd(a.energy + si, (double)v[0] * a.nu_third);
    __syncwarp();   // tables are rewritten by the next tile
}

__device__ __forceinline__ bool needs_mask(const TripArgs &a, uint32_t kb, uint32_t ib, uint32_t jb) {
    return kb == ib || ib == jb || (int64_t)(kb + 1) * 32 > a.n;
}

__device__ __forceinline__ void run_tile(const TripArgs &a, WarpSmem &sm, uint32_t kb, uint32_t ib, uint32_t jb,
                                         Acc &acc) {
    const int lane = threadIdx.x & 31;
    const bool new_pq = !acc.live || acc.kb != kb || acc.ib != ib;
    if (new_pq) flush_pq(a, acc, lane);
    if (needs_mask(a, kb, ib, jb))
        tile<true>(a, sm, kb, ib, jb, new_pq, acc);
    else
        tile<false>(a, sm, kb, ib, jb, new_pq, acc);
}

constexpr int kWarps = 2;          // 2 x 10 KB of tables per CTA

template <int STRAT>
__global__ void __launch_bounds__(32 * kWarps, 16 / kWarps) triplet32_kernel(TripArgs a) {
    __shared__ __align__(16) WarpSmem smem[kWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem &sm = smem[warp];
    Acc acc;
    acc.ep = acc.eq = 0.0;
    acc.kb = acc.ib = 0;
    acc.live = false;
    if (STRAT == TRI_BB) {
        const uint32_t jb = blockIdx.x * kWarps + warp, ib = blockIdx.y, kb = blockIdx.z;
        if (jb > ib || ib > kb) return;                  // outside the tetrahedron (warp-uniform)
        run_tile(a, sm, kb, ib, jb, acc);
    } else if (STRAT == TRI_LAMBDA) {
        const uint64_t w = a.omega_begin + ((uint64_t)blockIdx.y * gridDim.x + blockIdx.x) * kWarps + warp;
        if (w >= a.omega_end) return;
        uint32_t ib, jb, kb;
        tri::tet_map(w, ib, jb, kb);
        run_tile(a, sm, kb, ib, jb, acc);
    } else {
        // contiguous omega chunk per warp: consecutive tiles share (k, i)
        const uint64_t nb = a.omega_end - a.omega_begin;
        const uint64_t nw = (uint64_t)gridDim.x * kWarps;
        const uint64_t per = (nb + nw - 1) / nw;
        const uint64_t w0 = a.omega_begin + per * ((uint64_t)blockIdx.x * kWarps + warp);
        uint64_t w1 = w0 + per;
        if (w1 > a.omega_end) w1 = a.omega_end;
        if (w0 >= w1) return;
        uint32_t ib, jb, kb;
        tri::tet_map(w0, ib, jb, kb);
#pragma unroll 1
        for (uint64_t w = w0; w < w1; ++w) {
            run_tile(a, sm, kb, ib, jb, acc);
            if (++jb > ib) { jb = 0; if (++ib > kb) { ib = 0; ++kb; } }   // Eq. 1 successor
        }
    }
    flush_pq(a, acc, lane);
}

tri_status launch(const tet_map_t &m, int strategy, TripArgs a, cudaStream_t st) {
    const unsigned thr = 32 * kWarps;
    if (strategy == TRI_BB) {
        if (m.world > 1 || m.m > 65535) return TRI_ENOTSUP;
        const unsigned mm = (unsigned)m.m;
        triplet32_kernel<TRI_BB><<<dim3((mm + kWarps - 1) / kWarps, mm, mm), thr, 0, st>>>(a);
    } else if (strategy == TRI_LAMBDA) {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        triplet32_kernel<TRI_LAMBDA><<<tri::tile_grid((nb + kWarps - 1) / kWarps), thr, 0, st>>>(a);
    } else {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, triplet32_kernel<TRI_LAMBDA_PERSIST>, thr, 0);
        uint64_t g = (uint64_t)tri::sm_count() * (uint64_t)(per_sm > 0 ? per_sm : 1);
        if (g * kWarps > nb) g = (nb + kWarps - 1) / kWarps;
        triplet32_kernel<TRI_LAMBDA_PERSIST><<<(unsigned)g, thr, 0, st>>>(a);
    }
    tri::note_launches(1);
    return tri::cuda_status();
}

}  // namespace t32

}  // namespace

namespace tri {

tri_status launch_triplet(const tet_map_t &m, int strategy, const float *pts, double nu, double *energy,
                          cudaStream_t st) {
    if (cudaMemsetAsync(energy, 0, (size_t)m.n * sizeof(double), st) != cudaSuccess) return TRI_ECUDA;
    TripArgs a;
    a.pts = (const float4 *)pts;
    a.n = m.n;
    a.nu_third = nu / 3.0;
    a.energy = energy;
    a.omega_begin = m.omega_begin;
    a.omega_end = m.omega_end;
    a.m = (uint32_t)m.m;
    switch (m.rho) {
        case 8: return launch_r<8>(m, strategy, a, st);
        case 16: return launch_r<16>(m, strategy, a, st);
        case 32: return t32::launch(m, strategy, a, st);
        default: return TRI_EINVAL;
    }
}

}  // namespace tri
