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
    const float r = rsqrtf(abc);
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
        default: return TRI_EINVAL;
    }
}

}  // namespace tri
