// edm.cu -- Euclidean distance matrix on the packed lower triangle
// (readings Q7/Q8), HBM-write bound.
//
// Tile = rho x rho cells, tile coordinate from lambda(omega) (Eq. 4) or the BB
// grid.  The packed Eq. 1 layout puts row i at T(i), so a tile's
// row segment starts at an arbitrary 4-byte offset.  To issue only aligned
// vector streaming stores, every aligned CW-float CHUNK of the output slice
// (CW = 4: 16 B; CW = 8 at rho = 256: 32 B, the sm_100 256-bit store) is owned
// by the tile that holds the chunk's first cell; the owner computes all CW
// cells even when they run past the tile edge (EDM is pointwise, so the
// neighbour cells are computable anywhere).
//
// rho = 128 (the bench): ownership is per aligned 128-BYTE LINE instead (OwnW), so
// every warp store is 4 whole L2 lines.  A 512-B store at a 16-B phase touches 5
// lines, 2 of them partially, and that alone costs the write stream ~20 %
// (tools/probes/line_align.cu: 7.18 vs 5.93 TB/s for the same tiles with constant
// data).  Interior tiles (bj + 1 < bi: every line stays inside its row) take the fast
// path edm_tile_interior_line: column points staged once per tile in shared memory as
// four rotated SoA copies (one aligned LDS.128 per coordinate per lane at any phase),
// row points as float4s, the tile's rows walked as 32 same-phase quads {x, 63-x, 64+x,
// 127-x} so one set of column loads serves 16 cells per lane, two cells per
// FADD2/FMUL2/FFMA2, rows at 32-bit offsets from one base pointer; 8 CTAs of 4 warps per
// SM.  Round 2: 1.39 -> 1.22-1.35 ms per step in the bench's sustained loop (n = 65536, 3-D;
// box-dependent) and 1.55 -> 1.2 ms for 4 features.  In that loop the board sits at its
// 1 kW power cap (SM clock ~1.5-1.6 GHz, sw_power_cap): the stores alone cost 0.85-1.0 J per
// launch (= torch fill_), the arithmetic ~0.3 J more (profiles/r02_edm_power.txt), so
// energy per cell, not the write pattern, sets the sustained rate; isolated launches take
// 1.18-1.22 ms (7.0-7.3 TB/s).  Measured and rejected: single rows with
// scalar math, rho = 256 tiles (octets: 28 % fewer instructions, yet slower), 4 CTAs of 8
// warps (faster isolated, 2-3 % slower sustained), 3 / 2 CTAs, other store cache hints.
//
// Other tile edges: interior tiles walk ROWS rows per warp, lane k owning chunk k
// (rho = 32 CW, so each warp store is one contiguous 512 B / 1 KB run); the row's
// chunk phase delta = (-T(i)) mod CW is warp-uniform, so every lane takes its CW
// columns from a (2 CW - 1)-column register window through a uniform branch; the row
// offset is advanced incrementally (T(i+1) = T(i) + i + 1) and the row point is
// broadcast by shuffle.  Tiles touching the diagonal (bj >= bi - 1) take a checked
// path that walks Eq. 1 across row ends and the slice end, honouring the same
// ownership unit.
#include "tri_common.cuh"

namespace {

struct EdmArgs {
    const float *pts;
    int64_t ld, n;
    uint64_t omega_begin, omega_end;
    int64_t tile_row_begin;
    uint64_t out_offset, out_cells;
    float *out;
    bool vec4;                    // 4 features with ld % 4 == 0 and 16-byte aligned points
};

constexpr int kEdmThreads = 256;
constexpr int kWarps = kEdmThreads / 32;
#ifndef TRI_EDM128_NT
#define TRI_EDM128_NT 128
#endif
#ifndef TRI_EDM128_CTAS
#define TRI_EDM128_CTAS 8
#endif
// CTA shape per tile edge: rho = 128 (the line-owned path) TRI_EDM128_NT threads, at most
// TRI_EDM128_CTAS CTAs per SM (register budget); the other edges 256 threads
template <int RHO> struct EdmT {
    static constexpr int NT = RHO == 128 ? TRI_EDM128_NT : kEdmThreads;
    static constexpr int CTAS = RHO == 128 ? TRI_EDM128_CTAS : 4;
};

// Chunk width (floats) per tile edge: rho = 256 uses 32-byte chunks and the
// sm_100 256-bit store (STG.E.ENL2.256, 1 KB per warp store), rho = 128 16-byte
// chunks (512 B); a launch uses one chunk width for all its tiles, so chunk
// ownership is consistent across tiles.
template <int RHO> struct ChunkW { static constexpr int CW = RHO == 256 ? 8 : 4; };

template <int DIM, int WN>
__device__ __forceinline__ float dist_w(const float (&p)[DIM], const float (&w)[DIM][WN], int t) {
    const float dx = p[0] - w[0][t];
    float d2 = dx * dx;
#pragma unroll
    for (int d = 1; d < DIM; ++d) {
        const float dd = p[d] - w[d][t];
        d2 = fmaf(dd, dd, d2);
    }
    return sqrt_approx(d2);
}

template <int DIM>
__device__ __forceinline__ float dist_gmem(const EdmArgs &a, int64_t i, int64_t j) {
    float d2 = 0.f;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
        const float dd = __ldg(a.pts + i * a.ld + d) - __ldg(a.pts + j * a.ld + d);
        d2 = d == 0 ? dd * dd : fmaf(dd, dd, d2);
    }
    return sqrt_approx(d2);
}

__device__ __forceinline__ void st_cs_v8(float *p, const float (&v)[8]) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

template <int CW>
__device__ __forceinline__ void store_chunk(float *dst, const float (&v)[CW]) {
    if constexpr (CW == 8) st_cs_v8(dst, v);
    else st_cs_v4(dst, v[0], v[1], v[2], v[3]);
}

// one lane's chunk at window offset D (the row's phase delta)
template <int DIM, int CW, int D>
__device__ __forceinline__ void chunk_at(const float (&p)[DIM], const float (&w)[DIM][2 * CW - 1], float *dst) {
    float v[CW];
#pragma unroll
    for (int e = 0; e < CW; ++e) v[e] = dist_w<DIM, 2 * CW - 1>(p, w, D + e);
    store_chunk<CW>(dst, v);
}

// warp-uniform dispatch on delta in [0, CW)
template <int DIM, int CW, int D = 0>
__device__ __forceinline__ void chunk_phase(int delta, const float (&p)[DIM], const float (&w)[DIM][2 * CW - 1],
                                            float *dst) {
    if (delta == D) {
        chunk_at<DIM, CW, D>(p, w, dst);
    } else if constexpr (D + 1 < CW) {
        chunk_phase<DIM, CW, D + 1>(delta, p, w, dst);
    }
}

// Interior tile: rows [r0, r0+RHO) x cols [c0, c0+RHO), c0 + RHO < r0.
// One warp per row segment: lane k owns chunk k (RHO = 32 CW).  VEC4 (4 features, rows
// 16-byte aligned -- the paper's x, y, z, w points): points are read as float4,
// the row point by one broadcast load instead of four shuffles.
template <int RHO, int DIM, bool VEC4 = false>
__device__ __forceinline__ void edm_tile_interior(const EdmArgs &a, int64_t r0, int64_t c0) {
    constexpr int CW = ChunkW<RHO>::CW, WN = 2 * CW - 1;
    static_assert(RHO == 32 * CW, "one chunk per lane per row");
    constexpr int ROWS = RHO / kWarps;            // rows per warp (<= 32)
    static_assert(ROWS <= 32, "row points are broadcast from one lane each");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t rbase = r0 + (int64_t)warp * ROWS;
    if (rbase >= a.n) return;
    float w[DIM][WN];
#pragma unroll
    for (int t = 0; t < WN; ++t) {
        const int64_t col = c0 + CW * lane + t;               // < r0: always a valid point
        if constexpr (VEC4) {                                  // 4 features, 16-B rows: one LDG.128
            const float4 q = __ldg(reinterpret_cast<const float4 *>(a.pts + col * a.ld));
            w[0][t] = q.x; w[1][t] = q.y; w[2][t] = q.z; w[3][t] = q.w;
        } else {
#pragma unroll
            for (int d = 0; d < DIM; ++d) w[d][t] = __ldg(a.pts + col * a.ld + d);
        }
    }
    float pr[DIM];
    if constexpr (!VEC4) {
        const int64_t rr = rbase + (lane < ROWS ? lane : 0);
        const bool in = rr < a.n;
#pragma unroll
        for (int d = 0; d < DIM; ++d) pr[d] = in ? __ldg(a.pts + rr * a.ld + d) : 0.f;
    }
    const int nrows = (int)((a.n - rbase) < ROWS ? (a.n - rbase) : ROWS);
    uint64_t s = tri::T2((uint64_t)rbase) + (uint64_t)c0 - a.out_offset;   // local start of row rbase
    float *base = a.out + CW * lane;
#pragma unroll 1
    for (int rr = 0; rr < nrows; ++rr) {
        float p[DIM];
        if constexpr (VEC4) {                                  // the row point: one broadcast LDG.128
            const float4 q = __ldg(reinterpret_cast<const float4 *>(a.pts + (rbase + rr) * a.ld));
            p[0] = q.x; p[1] = q.y; p[2] = q.z; p[3 % DIM] = q.w;
        } else {
#pragma unroll
            for (int d = 0; d < DIM; ++d) p[d] = __shfl_sync(0xffffffffu, pr[d], rr);
        }
        const int delta = (int)((0u - (uint32_t)s) & (uint32_t)(CW - 1));
        chunk_phase<DIM, CW>(delta, p, w, base + (s + (uint64_t)delta));
        s += (uint64_t)(rbase + rr + 1);               // T(i+1) = T(i) + i + 1
    }
}

// rho = 128 with TRI_EDM_LINE: ownership is per 128-byte LINE (32 floats) instead of per
// 16-byte chunk.  Every aligned line of the output slice is written by the tile-row
// segment holding its first cell, by one warp store per 4 lines, so no warp store
// straddles a line boundary (a 512-B store at a 16-B phase touches 5 lines, 2 of them
// partially; tools/probes/line_align.cu measures what that costs the write stream).
#ifndef TRI_EDM_LINE
#define TRI_EDM_LINE 1
#endif
template <int RHO> struct OwnW { static constexpr int OW = (RHO == 128 && TRI_EDM_LINE) ? 32 : ChunkW<RHO>::CW; };
constexpr int kLineCols = 160;        // staged columns c0 + t (t < 160) per rotation: lanes reach 4 (31 + 7) + 3
template <int DIM> struct LineSmem { static constexpr int FLOATS = 4 * DIM * kLineCols + 4 * 128; };

// One row quad of a line-owned interior tile: tile rows {x, 63 - x, 64 + x, 127 - x} share
// the line phase (T(r0 + y) = T(r0) + r0 y + T(y) with r0 = 0 mod 128, and T(y) mod 32 is
// the same on exactly these four y < 128), so one set of column loads serves 16 cells per
// lane.  FULL: all four rows inside the domain, else bit g of vmask says row g is.
template <int DIM, bool FULL, class Addr>
__device__ __forceinline__ void edm_line_quad(const float *rl, const float4 *rowp, int x, uint32_t s32, int vmask,
                                              const Addr &addr) {
    const int delta = (int)((0u - s32) & 31u);
    const float *src = rl + (delta & 3) * DIM * kLineCols + (delta & ~3);
    ulonglong2 w[DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d) w[d] = *reinterpret_cast<const ulonglong2 *>(src + d * kLineCols);
    const int rows[4] = {x, 63 - x, 64 + x, 127 - x};
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        if (!FULL && !((vmask >> g) & 1)) continue;
        const float4 pq = rowp[rows[g]];
        const float pv[4] = {pq.x, pq.y, pq.z, pq.w};
        unsigned long long a01 = 0, a23 = 0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
            unsigned long long e01, e23, pp;
            asm("mov.b64 %0, {%1, %1};" : "=l"(pp) : "f"(pv[d]));
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(e01) : "l"(pp), "l"(w[d].x));
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(e23) : "l"(pp), "l"(w[d].y));
            if (d == 0) {
                asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(a01) : "l"(e01));
                asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(a23) : "l"(e23));
            } else {
                asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(a01) : "l"(e01));
                asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(a23) : "l"(e23));
            }
        }
        float v[4];
        asm("mov.b64 {%0, %1}, %2;" : "=f"(v[0]), "=f"(v[1]) : "l"(a01));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(v[2]), "=f"(v[3]) : "l"(a23));
        st_cs_v4(addr(g, delta), sqrt_approx(v[0]), sqrt_approx(v[1]), sqrt_approx(v[2]), sqrt_approx(v[3]));
    }
}

// Interior tile, line ownership (rho = 128).  The row's line phase delta = (-T(i)) mod 32 =
// 4a + b is warp-uniform; lane k writes cells delta + 4k .. + 3 of the segment, i.e. columns
// c0 + 4(k + a) + b + e.  The tile's 163 column points are staged in shared memory as four
// rotated SoA copies rot[b][d][t] = point (c0 + t + b), so every lane reads its 4 columns of
// one coordinate with one aligned LDS.128 (a warp reads 512 contiguous bytes: 4 wavefronts),
// and the tile's 128 row points as float4s (one broadcast LDS.128 per row).  The 128 rows
// fall into 32 classes of four with the same phase (edm_line_quad), so a warp walks four
// row QUADS: one set of column loads serves 16 cells per lane.
template <int DIM, bool VEC4 = false>
__device__ __forceinline__ void edm_tile_interior_line(const EdmArgs &a, int64_t r0, int64_t c0, float *rot) {
    constexpr int RHO = 128;
    float4 *rowp = reinterpret_cast<float4 *>(rot + 4 * DIM * kLineCols);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();                                          // the previous tile's readers are done
    for (int t = threadIdx.x; t < kLineCols + 3 + RHO; t += EdmT<RHO>::NT) {
        const bool is_col = t < kLineCols + 3;
        const int64_t pt = is_col ? c0 + t : r0 + (t - kLineCols - 3);   // col <= c0 + 162 < r0
        if (!is_col && pt >= a.n) continue;
        float q[4] = {0.f, 0.f, 0.f, 0.f};
        if constexpr (VEC4) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(a.pts + pt * a.ld));
            q[0] = v.x; q[1] = v.y; q[2] = v.z; q[3] = v.w;
        } else {
#pragma unroll
            for (int d = 0; d < DIM; ++d) q[d] = __ldg(a.pts + pt * a.ld + d);
        }
        if (is_col) {
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (t - b >= 0 && t - b < kLineCols) {
#pragma unroll
                    for (int d = 0; d < DIM; ++d) rot[(b * DIM + d) * kLineCols + t - b] = q[d];
                }
        } else {
            rowp[t - kLineCols - 3] = make_float4(q[0], q[1], q[2], q[3]);
        }
    }
    __syncthreads();
    // warp w takes x = XW w .. XW w + XW - 1 (XW = 32 / warps): rows {x, 63 - x, 64 + x, 127 - x},
    // all 128 rows over the CTA's warps
    constexpr int XW = 32 / (EdmT<128>::NT / 32);
    const int x0 = XW * warp;
    const float *rl = rot + 4 * lane;
    const bool full = r0 + 127 < a.n;
    const uint32_t u0 = (uint32_t)r0;
    const uint64_t s0 = tri::T2((uint64_t)r0) + (uint64_t)c0 - a.out_offset;   // local start of row r0
    auto vmask_of = [&](int x) {
        return (int)(r0 + x < a.n) | ((int)(r0 + 63 - x < a.n) << 1) | ((int)(r0 + 64 + x < a.n) << 2) |
               ((int)(r0 + 127 - x < a.n) << 3);
    };
    if (r0 < (int64_t)(1 << 25)) {
        // rows r0 + y at 32-bit offsets T(r0 + y) - T(r0) = r0 y + T(y) < 2^32 from one 64-bit base:
        // one IMAD.WIDE per store address, one IADD3 per row step
        float *const B = a.out + s0 + 4 * lane;
        const int ys[4] = {x0, 63 - x0, 64 + x0, 127 - x0};
        uint32_t o[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) o[g] = u0 * (uint32_t)ys[g] + (uint32_t)(ys[g] * (ys[g] + 1) / 2);
        const uint32_t sp = (uint32_t)s0;
        auto addr = [&](int g, int delta) { return (B + delta) + o[g]; };
        auto step = [&](int x) {
            o[0] += u0 + (uint32_t)x + 1u;                // T(i + 1) - T(i) = i + 1
            o[1] -= u0 + 63u - (uint32_t)x;               // T(i - 1) - T(i) = -i
            o[2] += u0 + 65u + (uint32_t)x;
            o[3] -= u0 + 127u - (uint32_t)x;
        };
        if (full) {
#pragma unroll
            for (int t = 0; t < XW; ++t) {
                edm_line_quad<DIM, true>(rl, rowp, x0 + t, sp + o[0], 15, addr);
                step(x0 + t);
            }
        } else {
#pragma unroll 1
            for (int t = 0; t < XW; ++t) {
                const int vmask = vmask_of(x0 + t);
                if (vmask) edm_line_quad<DIM, false>(rl, rowp, x0 + t, sp + o[0], vmask, addr);
                step(x0 + t);
            }
        }
    } else {                                              // very large n: 64-bit row pointers
        const int64_t rr0[4] = {r0 + x0, r0 + 63 - x0, r0 + 64 + x0, r0 + 127 - x0};
        float *pr[4];
#pragma unroll
        for (int g = 0; g < 4; ++g)
            pr[g] = a.out + (tri::T2((uint64_t)rr0[g]) + (uint64_t)c0 - a.out_offset) + 4 * lane;
        uint32_t s32 = (uint32_t)(tri::T2((uint64_t)rr0[0]) + (uint64_t)c0 - a.out_offset);   // phase bits
        auto addr = [&](int g, int delta) { return pr[g] + delta; };
#pragma unroll 1
        for (int t = 0; t < XW; ++t) {
            const int x = x0 + t;
            const int vmask = vmask_of(x);
            if (vmask) edm_line_quad<DIM, false>(rl, rowp, x, s32, vmask, addr);
            pr[0] += u0 + (uint32_t)x + 1u;
            pr[1] -= u0 + 63u - (uint32_t)x;
            pr[2] += u0 + 65u + (uint32_t)x;
            pr[3] -= u0 + 127u - (uint32_t)x;
            s32 += u0 + (uint32_t)x + 1u;
        }
    }
}

// Any tile (used for tiles touching the diagonal, and for rho < 128): every
// chunk slot of every row, cells walked along Eq. 1, all bounds checked.  A slot belongs
// to this segment when its ownership unit (OW floats: the chunk, or the 128-B line at
// rho = 128) starts inside the segment; it may run past the segment / row end.
template <int RHO, int DIM>
__device__ __forceinline__ void edm_tile_checked(const EdmArgs &a, int64_t r0, int64_t c0) {
    constexpr int CW = ChunkW<RHO>::CW, OW = OwnW<RHO>::OW;
    constexpr int L = RHO / CW;                       // chunk slots per row segment
    const int t = threadIdx.x;
#pragma unroll 1
    for (int q = t; q < RHO * L; q += EdmT<RHO>::NT) {
        const int rr = q / L, k = q % L;
        const int64_t i = r0 + rr;
        if (i >= a.n) break;
        const uint64_t s = tri::T2((uint64_t)i) + (uint64_t)c0 - a.out_offset;
        const int64_t seg = i - c0 + 1;
        const int64_t len = seg < RHO ? seg : RHO;
        const int dl = (int)((0u - (uint32_t)s) & (uint32_t)(OW - 1));
        const int off = dl + CW * k;
        if (dl + (CW * k / OW) * OW >= len) continue;  // unit owned by the next segment
        const uint64_t c = s + (uint64_t)off;
        float v[CW];
        int64_t ii = i, jj = c0 + off;
#pragma unroll
        for (int e = 0; e < CW; ++e) {
            while (jj > ii) { jj -= ii + 1; ++ii; }
            v[e] = (c + e < a.out_cells && ii < a.n) ? dist_gmem<DIM>(a, ii, jj) : 0.f;
            ++jj;
        }
        float *dst = a.out + c;
        if (c + CW <= a.out_cells) {
            store_chunk<CW>(dst, v);
        } else {
#pragma unroll
            for (int e = 0; e < CW; ++e)
                if (c + e < a.out_cells) dst[e] = v[e];
        }
    }
}

template <int RHO, int DIM>
__device__ __forceinline__ void edm_tile(const EdmArgs &a, uint32_t bi, uint32_t bj, float *rot) {
    const int64_t r0 = (int64_t)bi * RHO, c0 = (int64_t)bj * RHO;
    if constexpr (OwnW<RHO>::OW == 32) {
        if (bj + 1 < bi) {
            if (DIM == 4 && a.vec4) edm_tile_interior_line<DIM, DIM == 4>(a, r0, c0, rot);
            else edm_tile_interior_line<DIM>(a, r0, c0, rot);
            return;
        }
    } else if constexpr (RHO >= 128) {
        if (bj + 1 < bi) {
            if (DIM == 4 && a.vec4) edm_tile_interior<RHO, DIM, DIM == 4>(a, r0, c0);
            else edm_tile_interior<RHO, DIM>(a, r0, c0);
            return;
        }
    }
    edm_tile_checked<RHO, DIM>(a, r0, c0);
}

template <int RHO, int DIM, int STRAT>
__global__ void __launch_bounds__(EdmT<RHO>::NT, EdmT<RHO>::CTAS) edm_kernel(EdmArgs a) {
    __shared__ __align__(16) float rot[OwnW<RHO>::OW == 32 ? LineSmem<DIM>::FLOATS : 4];
    if (STRAT == TRI_BB) {
        const uint32_t bj = blockIdx.x;
        const uint32_t bi = blockIdx.y + (uint32_t)a.tile_row_begin;
        if (bj > bi) return;                                  // discard
        edm_tile<RHO, DIM>(a, bi, bj, rot);
    } else if (STRAT == TRI_LAMBDA) {
        const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (w >= a.omega_end) return;
        uint32_t bi, bj;
        tri::lambda_map(w, bi, bj);
        edm_tile<RHO, DIM>(a, bi, bj, rot);
    } else if (STRAT == TRI_LAMBDA_CLC) {
        __shared__ tri::ClcSched clc;
        if (threadIdx.x == 0) clc.init();
        __syncthreads();
        uint32_t bx = blockIdx.x, by = blockIdx.y, phase = 0;
#pragma unroll 1
        while (true) {
            if (threadIdx.x == 0) clc.request();              // overlaps the tile below
            const uint64_t w = a.omega_begin + (uint64_t)by * gridDim.x + bx;
            if (w < a.omega_end) {
                uint32_t bi, bj;
                tri::lambda_map(w, bi, bj);
                edm_tile<RHO, DIM>(a, bi, bj, rot);
            }
            const bool more = clc.receive(phase, bx, by);
            __syncthreads();                                  // handle read by all before the next request
            if (!more) break;
        }
    } else {
#pragma unroll 1
        for (tri::TileWalk t(a.omega_begin, a.omega_end); t.more(); t.next()) edm_tile<RHO, DIM>(a, t.bi, t.bj, rot);
    }
}

template <int RHO, int DIM>
tri_status launch_rd(const tri_map_t &m, int strategy, EdmArgs a, cudaStream_t st) {
    if (strategy == TRI_BB) {
        const int64_t tr0 = m.row_begin / m.rho;
        const int64_t tr1 = (m.row_end + m.rho - 1) / m.rho;
        if (tr1 <= tr0) return TRI_OK;
        if (tr1 - tr0 > 65535) return TRI_ENOTSUP;
        a.tile_row_begin = tr0;
        edm_kernel<RHO, DIM, TRI_BB><<<dim3((unsigned)m.m, (unsigned)(tr1 - tr0)), EdmT<RHO>::NT, 0, st>>>(a);
    } else if (strategy == TRI_LAMBDA) {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        edm_kernel<RHO, DIM, TRI_LAMBDA><<<tri::tile_grid(nb), EdmT<RHO>::NT, 0, st>>>(a);
    } else if (strategy == TRI_LAMBDA_CLC) {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        edm_kernel<RHO, DIM, TRI_LAMBDA_CLC><<<tri::tile_grid(nb), EdmT<RHO>::NT, 0, st>>>(a);
    } else {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, edm_kernel<RHO, DIM, TRI_LAMBDA_PERSIST>,
                                                      EdmT<RHO>::NT, 0);
        uint64_t g = (uint64_t)tri::sm_count() * (uint64_t)(per_sm > 0 ? per_sm : 1);
        if (g > nb) g = nb;
        edm_kernel<RHO, DIM, TRI_LAMBDA_PERSIST><<<(unsigned)g, EdmT<RHO>::NT, 0, st>>>(a);
    }
    tri::note_launches(1);
    return tri::cuda_status();
}

template <int RHO>
tri_status launch_r(const tri_map_t &m, int strategy, int dim, EdmArgs a, cudaStream_t st) {
    switch (dim) {
        case 1: return launch_rd<RHO, 1>(m, strategy, a, st);
        case 2: return launch_rd<RHO, 2>(m, strategy, a, st);
        case 3: return launch_rd<RHO, 3>(m, strategy, a, st);
        default: return launch_rd<RHO, 4>(m, strategy, a, st);
    }
}

}  // namespace

namespace tri {

tri_status launch_edm(const tri_map_t &m, int strategy, const float *pts, int dim, int64_t ld, float *out,
                      cudaStream_t st) {
    EdmArgs a;
    a.pts = pts; a.ld = ld; a.n = m.n;
    a.omega_begin = m.omega_begin; a.omega_end = m.omega_end;
    a.tile_row_begin = 0;
    a.out_offset = m.out_offset; a.out_cells = m.out_cells;
    a.out = out;
    a.vec4 = dim == 4 && (ld & 3) == 0 && (((uintptr_t)pts) & 15u) == 0;
    switch (m.rho) {
        case 32: return launch_r<32>(m, strategy, dim, a, st);
        case 64: return launch_r<64>(m, strategy, dim, a, st);
        case 128: return launch_r<128>(m, strategy, dim, a, st);
        default: return launch_r<256>(m, strategy, dim, a, st);
    }
}

}  // namespace tri

// ---------------------------------------------------------------- host-buffer EDM
// Row bands (multiples of rho rows) are computed into a ping-pong device
// workspace and copied to the host buffer while the next band computes.
extern "C" tri_status tri_edm_host(const tri_map_t *map, int32_t strategy, const float *h_pts, int32_t dim,
                                   int64_t ld, size_t pts_bytes, float *d_pts_ws, size_t pts_ws_bytes,
                                   float *h_out, size_t out_bytes, void *d_ws, size_t ws_bytes,
                                   uint64_t band_cells) {
    using namespace tri;
    reset_launches();
    if (!h_pts || !d_pts_ws || !h_out || !d_ws) return TRI_EINVAL;
    // tri_edm's checks (map, strategy, rho, dim / ld, both capacities); RB has no band form
    if (strategy == TRI_RB || edm_args_bad(map, strategy, dim, ld, pts_bytes, out_bytes)) return TRI_EINVAL;
    if (pts_ws_bytes / 4u / (uint64_t)ld < (uint64_t)map->n || (((uintptr_t)d_pts_ws) & 15u)) return TRI_EINVAL;
    if (((uintptr_t)d_ws) & 31u) return TRI_EINVAL;
    if (map->out_cells == 0) return TRI_OK;
    {   // one tile row of the slice (the band granule) must fit a workspace half and band_cells
        const uint64_t half = (ws_bytes / 2 / 4) & ~7ull;
        const uint64_t lim = band_cells && band_cells < half ? (band_cells & ~7ull) : half;
        const uint64_t last = (uint64_t)map->row_end, first = last > (uint64_t)map->rho ? last - map->rho : 0;
        if (T2(last) - T2(first) > lim) return TRI_EINVAL;
    }
    uint64_t cap = (ws_bytes / 2 / 4) & ~7ull;          // floats per buffer, 32-byte multiple
    if (band_cells && band_cells < cap) cap = band_cells & ~7ull;
    const int64_t rho = map->rho;
    float *buf[2] = {(float *)d_ws, (float *)d_ws + ((ws_bytes / 2 / 4) & ~7ull)};
    cudaStream_t sc = nullptr, sx = nullptr;
    cudaEvent_t done_k[2] = {nullptr, nullptr}, done_c[2] = {nullptr, nullptr};
    tri_status rc = TRI_OK;
    int launches = 0;
    if (cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&sx, cudaStreamNonBlocking) != cudaSuccess) {
        rc = TRI_ECUDA;
    }
    for (int b = 0; b < 2 && rc == TRI_OK; ++b)
        if (cudaEventCreateWithFlags(&done_k[b], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&done_c[b], cudaEventDisableTiming) != cudaSuccess)
            rc = TRI_ECUDA;
    if (rc == TRI_OK &&
        cudaMemcpyAsync(d_pts_ws, h_pts, (size_t)(4ull * ((uint64_t)(map->n - 1) * (uint64_t)ld + (uint64_t)dim)),
                        cudaMemcpyHostToDevice, sc) !=
            cudaSuccess)
        rc = TRI_ECUDA;
    int64_t ra = map->row_begin;
    int band = 0;
    while (rc == TRI_OK && ra < map->row_end) {
        int64_t rb = ra + rho;
        if (rb > map->row_end) rb = map->row_end;
        while (rb < map->row_end) {
            int64_t nx = rb + rho > map->row_end ? map->row_end : rb + rho;
            if (T2((uint64_t)nx) - T2((uint64_t)ra) > cap) break;
            rb = nx;
        }
        const uint64_t cells = T2((uint64_t)rb) - T2((uint64_t)ra);
        if (cells > cap) { rc = TRI_EINVAL; break; }
        tri_map_t bm = *map;
        bm.row_begin = ra; bm.row_end = rb;
        bm.omega_begin = T2((uint64_t)(ra / rho));
        bm.omega_end = T2((uint64_t)((rb + rho - 1) / rho));
        bm.out_offset = T2((uint64_t)ra);
        bm.out_cells = cells;
        const int slot = band & 1;
        if (band >= 2) cudaStreamWaitEvent(sc, done_c[slot], 0);
        rc = launch_edm(bm, strategy, d_pts_ws, dim, ld, buf[slot], sc);
        if (rc != TRI_OK) break;
        ++launches;
        cudaEventRecord(done_k[slot], sc);
        cudaStreamWaitEvent(sx, done_k[slot], 0);
        if (cudaMemcpyAsync(h_out + (bm.out_offset - map->out_offset), buf[slot], cells * 4u,
                            cudaMemcpyDeviceToHost, sx) != cudaSuccess) {
            rc = TRI_ECUDA;
            break;
        }
        cudaEventRecord(done_c[slot], sx);
        ra = rb;
        ++band;
    }
    if (sc && cudaStreamSynchronize(sc) != cudaSuccess) rc = TRI_ECUDA;
    if (sx && cudaStreamSynchronize(sx) != cudaSuccess) rc = TRI_ECUDA;
    for (int b = 0; b < 2; ++b) {
        if (done_k[b]) cudaEventDestroy(done_k[b]);
        if (done_c[b]) cudaEventDestroy(done_c[b]);
    }
    if (sc) cudaStreamDestroy(sc);
    if (sx) cudaStreamDestroy(sx);
    (void)launches;
    return rc;
}
