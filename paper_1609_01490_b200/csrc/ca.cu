// ca.cu -- one generation of Life B3/S23 on the triangular domain
// {(i, j): 0 <= j <= i < n} (P:79-80 names cellular automata on triangular
// domains, citing Conway's Life; cells outside the triangle are dead --
// DESIGN.md reading Q11).  State: u8 {0,1} in the packed Eq. 1 layout.
//
// Block-space mapping: a rho x rho tile from lambda(omega) or the
// BB grid; inside the tile, every aligned 16-byte CHUNK of the output slice is
// owned by the tile holding its first cell (as in edm.cu), so all stores are
// aligned 16-byte streaming stores.  A chunk's 16 cells need the 18-byte
// windows of rows i-1, i, i+1; each window is read as six aligned 32-bit words
// (L1-resident: neighbouring lanes and rows share lines) and realigned with
// funnel shifts.  The rule is evaluated 4 cells per 32-bit word (SWAR):
// vertical byte sums of the three rows first (<= 3 per byte), then the
// horizontal 3-sum (<= 9, incl. self), then B3/S23 as bit-plane logic:
//   next = (sum9 == 3) | (self & (sum9 == 4)).
// Every chunk runs the same SIMT code: interior chunks load unmasked; chunks
// touching column -1, the diagonal or the slice edge load with byte masks
// (columns outside [0, r] of row r and absent rows read as dead); a chunk that
// crosses the end of row i is two 16-cell evaluations (row i at j0, row i+1 at
// j0 - i - 1) merged bytewise.  Only rows i < 16 (chunks spanning 3+ rows)
// fall back to a per-cell loop.
#include "tri_common.cuh"

namespace {

struct CaArgs {
    const uint8_t *in;
    uint8_t *out;
    const uint8_t *above, *below;  // halo rows R0-1 and R1 (NULL = dead)
    int64_t n, R0, R1;             // this slice owns rows [R0, R1)
    uint64_t base;                 // T(R0)
    uint64_t out_cells;
    uint64_t omega_begin, omega_end;
    int64_t tile_row_begin;
};

// Row pointer to column 0 of row r, or nullptr for a dead row.
__device__ __forceinline__ const uint8_t *row_ptr(const CaArgs &a, int64_t r) {
    if (r < 0 || r >= a.n) return nullptr;
    if (r < a.R0) return (r == a.R0 - 1) ? a.above : nullptr;
    if (r >= a.R1) return (r == a.R1) ? a.below : nullptr;
    return a.in + (tri::T2((uint64_t)r) - a.base);
}

__device__ __forceinline__ uint32_t cell(const CaArgs &a, int64_t r, int64_t c) {
    if (c < 0 || c > r) return 0;
    const uint8_t *p = row_ptr(a, r);
    return p ? (uint32_t)p[c] : 0u;
}

__device__ __forceinline__ uint32_t life_cell(const CaArgs &a, int64_t i, int64_t j) {
    uint32_t nb = 0;
#pragma unroll
    for (int di = -1; di <= 1; ++di)
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj)
            if (di || dj) nb += cell(a, i + di, j + dj);
    const uint32_t self = cell(a, i, j);
    return (nb == 3u) | (self & (nb == 2u));
}

// Window of row r, columns [cs, cs + 18): X[t] = bytes of columns cs+4t .. cs+4t+3.
// MASK: columns outside [0, r] read as 0 and words holding no valid column are
// never loaded (so nothing outside the row's buffer is touched).
template <bool MASK>
__device__ __forceinline__ void window(const CaArgs &a, int64_t r, int64_t cs, uint32_t (&X)[5]) {
    const uint8_t *p = MASK ? row_ptr(a, r) : a.in + (tri::T2((uint64_t)r) - a.base);
    if (MASK && !p) {                       // dead row (outside the domain / absent halo)
#pragma unroll
        for (int t = 0; t < 5; ++t) X[t] = 0;
        return;
    }
    const uintptr_t ad = (uintptr_t)(p + cs);
    const uint32_t sh = (uint32_t)(ad & 3u);
    const uint32_t *w = (const uint32_t *)(ad & ~(uintptr_t)3);
    uint32_t R[6];
#pragma unroll
    for (int t = 0; t < 6; ++t) {
        if (MASK) {
            const int64_t cw = cs - (int64_t)sh + 4 * t;       // column of the word's byte 0
            if (cw + 3 < 0 || cw > r) {
                R[t] = 0;
            } else {
                uint32_t v = __ldg(w + t);
                const int lo = cw < 0 ? (int)(-cw) : 0;
                const int hi = cw + 3 > r ? (int)(cw + 3 - r) : 0;
                v &= (0xffffffffu << (8 * lo)) & (0xffffffffu >> (8 * hi));
                R[t] = v;
            }
        } else {
            R[t] = __ldg(w + t);
        }
    }
#pragma unroll
    for (int t = 0; t < 5; ++t) X[t] = __funnelshift_r(R[t], R[t + 1], 8 * sh);
}

__device__ __forceinline__ uint32_t life_word(uint32_t sum9, uint32_t self) {
    // bytes of sum9 are 0..9 (4 bits).  Bit planes at bit 0 of every byte:
    const uint32_t b0 = sum9, b1 = sum9 >> 1, b2 = sum9 >> 2, b3 = sum9 >> 3;
    const uint32_t is3 = ~b3 & ~b2 & b1 & b0;
    const uint32_t is4 = ~b3 & b2 & ~b1 & ~b0;
    return (is3 | (self & is4)) & 0x01010101u;
}

// Next state of the 16 cells (r, js .. js+15) into o[4] (byte q = cell js+q).
template <bool MASK>
__device__ __forceinline__ void eval16(const CaArgs &a, int64_t r, int64_t js, uint32_t (&o)[4]) {
    uint32_t U[5], M[5], D[5], V[5];
    window<MASK>(a, r - 1, js - 1, U);
    window<MASK>(a, r, js - 1, M);
    window<MASK>(a, r + 1, js - 1, D);
#pragma unroll
    for (int t = 0; t < 5; ++t) V[t] = U[t] + M[t] + D[t];       // vertical 3-sums
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const uint32_t sum9 = V[w] + __funnelshift_r(V[w], V[w + 1], 8) + __funnelshift_r(V[w], V[w + 1], 16);
        const uint32_t self = __funnelshift_r(M[w], M[w + 1], 8);
        o[w] = life_word(sum9, self);
    }
}

__device__ __forceinline__ void store_chunk(const CaArgs &a, uint64_t c, const uint32_t (&o)[4]) {
    uint8_t *dst = a.out + c;
    if (c + 16 <= a.out_cells) {
        st_cs_v4u(dst, o[0], o[1], o[2], o[3]);
    } else {
#pragma unroll 1
        for (int q = 0; q < 16; ++q)
            if (c + q < a.out_cells) dst[q] = (uint8_t)(o[q >> 2] >> (8 * (q & 3)));
    }
}

template <int RHO>
__device__ __forceinline__ void ca_tile(const CaArgs &a, uint32_t bi, uint32_t bj) {
    constexpr int L = RHO / 16;                 // chunk lanes per row segment
    constexpr int RPW = 32 / L;                 // rows per warp pass
    constexpr int NW = 8;
    constexpr int ROWS_PER_WARP = RHO / NW;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = lane % L, rs = lane / L;
    const int64_t r0 = (int64_t)bi * RHO, c0 = (int64_t)bj * RHO;
    const int64_t rbase = r0 + (int64_t)warp * ROWS_PER_WARP;
#pragma unroll 1
    for (int rr = rs; rr < ROWS_PER_WARP; rr += RPW) {
        const int64_t i = rbase + rr;
        if (i >= a.R1) break;
        if (i < a.R0) continue;
        const uint64_t s = tri::T2((uint64_t)i) + (uint64_t)c0 - a.base;   // local segment start
        const int64_t seg = i - c0 + 1;
        const int64_t len = seg < RHO ? seg : RHO;
        const int delta = (int)((0u - (uint32_t)s) & 15u);
        const int off = delta + 16 * k;
        if (off >= len) continue;
        const uint64_t c = s + (uint64_t)off;
        const int64_t j0 = c0 + off;              // first cell column
        uint32_t o[4];
        if (j0 >= 1 && j0 + 16 <= i - 1 && i > a.R0 && i + 1 < a.R1) {
            eval16<false>(a, i, j0, o);           // interior: all window rows/columns in the slice
        } else if (j0 + 15 <= i) {
            eval16<true>(a, i, j0, o);            // touches column -1 / the diagonal
        } else if (i >= 16) {
            // crosses the row end: cells j0..i of row i, then 0.. of row i+1
            uint32_t A[4], B[4];
            const int na = (int)(i - j0 + 1);     // 1..15 cells from row i
            eval16<true>(a, i, j0, A);
            eval16<true>(a, i + 1, j0 - i - 1, B);
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const int lo = na - 4 * w;        // bytes of word w taken from A
                const uint32_t m = lo >= 4 ? 0xffffffffu : (lo <= 0 ? 0u : (0xffffffffu >> (8 * (4 - lo))));
                o[w] = (A[w] & m) | (B[w] & ~m);
            }
        } else {
            // rows < 16: a chunk may span several rows -- per cell along Eq. 1
            o[0] = o[1] = o[2] = o[3] = 0;
            int64_t ii = i, jj = j0;
#pragma unroll 1
            for (int q = 0; q < 16; ++q) {
                while (jj > ii) { jj -= ii + 1; ++ii; }
                if (c + q < a.out_cells) o[q >> 2] |= life_cell(a, ii, jj) << (8 * (q & 3));
                ++jj;
            }
        }
        store_chunk(a, c, o);
    }
}

constexpr int kCaThreads = 256;

template <int RHO, int STRAT>
__global__ void __launch_bounds__(kCaThreads) ca_kernel(CaArgs a) {
    if (STRAT == TRI_BB) {
        const uint32_t bj = blockIdx.x;
        const uint32_t bi = blockIdx.y + (uint32_t)a.tile_row_begin;
        if (bj > bi) return;
        ca_tile<RHO>(a, bi, bj);
    } else if (STRAT == TRI_LAMBDA) {
        const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (w >= a.omega_end) return;
        uint32_t bi, bj;
        tri::lambda_map(w, bi, bj);
        ca_tile<RHO>(a, bi, bj);
    } else {
#pragma unroll 1
        for (uint64_t w = a.omega_begin + blockIdx.x; w < a.omega_end; w += gridDim.x) {
            uint32_t bi, bj;
            tri::lambda_map(w, bi, bj);
            ca_tile<RHO>(a, bi, bj);
        }
    }
}

template <int RHO>
tri_status launch_r(const tri_map_t &m, int strategy, CaArgs a, cudaStream_t st) {
    if (strategy == TRI_BB) {
        const int64_t tr0 = m.row_begin / m.rho;
        const int64_t tr1 = (m.row_end + m.rho - 1) / m.rho;
        if (tr1 <= tr0) return TRI_OK;
        if (tr1 - tr0 > 65535) return TRI_ENOTSUP;
        a.tile_row_begin = tr0;
        ca_kernel<RHO, TRI_BB><<<dim3((unsigned)m.m, (unsigned)(tr1 - tr0)), kCaThreads, 0, st>>>(a);
    } else if (strategy == TRI_LAMBDA) {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        ca_kernel<RHO, TRI_LAMBDA><<<tri::tile_grid(nb), kCaThreads, 0, st>>>(a);
    } else {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ca_kernel<RHO, TRI_LAMBDA_PERSIST>, kCaThreads, 0);
        uint64_t g = (uint64_t)tri::sm_count() * (uint64_t)(per_sm > 0 ? per_sm : 1);
        if (g > nb) g = nb;
        ca_kernel<RHO, TRI_LAMBDA_PERSIST><<<(unsigned)g, kCaThreads, 0, st>>>(a);
    }
    tri::note_launches(1);
    return tri::cuda_status();
}

}  // namespace

namespace tri {

tri_status launch_ca(const tri_map_t &m, int strategy, const uint8_t *in, uint8_t *out, const uint8_t *above,
                     const uint8_t *below, cudaStream_t st) {
    if (((uintptr_t)out & 15u) != 0 || ((uintptr_t)in & 15u) != 0) return TRI_EINVAL;
    CaArgs a;
    a.in = in; a.out = out;
    a.above = m.row_begin > 0 ? above : nullptr;
    a.below = m.row_end < m.n ? below : nullptr;
    a.n = m.n; a.R0 = m.row_begin; a.R1 = m.row_end;
    a.base = m.out_offset; a.out_cells = m.out_cells;
    a.omega_begin = m.omega_begin; a.omega_end = m.omega_end;
    a.tile_row_begin = 0;
    switch (m.rho) {
        case 128: return launch_r<128>(m, strategy, a, st);
        case 256: return launch_r<256>(m, strategy, a, st);
        case 512: return launch_r<512>(m, strategy, a, st);
        default: return TRI_EINVAL;
    }
}

}  // namespace tri
