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
// horizontal byte sums of each row (<= 3 per byte), vertical sum (<= 9, incl.
// self), then B3/S23 as bit-plane logic:
//   next = (sum9 == 3) | (self & (sum9 == 4)).
// Chunks whose window touches the triangle's edge (column -1, the diagonal),
// a row end, or the slice end take a per-cell path with explicit bounds.
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

// Horizontal sums of an 18-byte window (cols c-1 .. c+16) of one row.
// R: six aligned words covering the window, sh: byte offset of col c-1 in R[0].
// H[w] = bytes (cols 4w+c-1 + cols 4w+c + cols 4w+c+1) for the 4 cells of word w,
// M[w] = the row's own cells 4w+c .. 4w+c+3.
__device__ __forceinline__ void row_sums(const uint32_t (&R)[6], uint32_t sh, uint32_t (&H)[4],
                                         uint32_t (&M)[4]) {
    uint32_t X[5];
#pragma unroll
    for (int t = 0; t < 5; ++t) X[t] = __funnelshift_r(R[t], R[t + 1], 8 * sh);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const uint32_t mid = __funnelshift_r(X[w], X[w + 1], 8);
        const uint32_t rgt = __funnelshift_r(X[w], X[w + 1], 16);
        H[w] = X[w] + mid + rgt;
        M[w] = mid;
    }
}

__device__ __forceinline__ void load6(const uint8_t *row, int64_t c_left, uint32_t (&R)[6], uint32_t &sh) {
    if (!row) {
#pragma unroll
        for (int t = 0; t < 6; ++t) R[t] = 0;
        sh = 0;
        return;
    }
    const uintptr_t ad = (uintptr_t)(row + c_left);
    sh = (uint32_t)(ad & 3u);
    const uint32_t *w = (const uint32_t *)(ad & ~(uintptr_t)3);
#pragma unroll
    for (int t = 0; t < 6; ++t) R[t] = __ldg(w + t);
}

__device__ __forceinline__ uint32_t life_word(uint32_t sum9, uint32_t self) {
    // bytes of sum9 are 0..9 (4 bits).  Bit planes at bit 0 of every byte:
    const uint32_t b0 = sum9, b1 = sum9 >> 1, b2 = sum9 >> 2, b3 = sum9 >> 3;
    const uint32_t is3 = ~b3 & ~b2 & b1 & b0;
    const uint32_t is4 = ~b3 & b2 & ~b1 & ~b0;
    return (is3 | (self & is4)) & 0x01010101u;
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
        uint8_t *dst = a.out + c;
        if (j0 >= 1 && j0 + 16 <= i - 1) {
            // all 18 window columns valid in rows i-1, i, i+1
            uint32_t R[6], sh, Hu[4], Hm[4], Hd[4], Mu[4], Mm[4], Md[4];
            load6(row_ptr(a, i - 1), j0 - 1, R, sh);
            row_sums(R, sh, Hu, Mu);
            load6(row_ptr(a, i), j0 - 1, R, sh);
            row_sums(R, sh, Hm, Mm);
            load6(row_ptr(a, i + 1), j0 - 1, R, sh);
            row_sums(R, sh, Hd, Md);
            uint32_t o[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) o[w] = life_word(Hu[w] + Hm[w] + Hd[w], Mm[w]);
            st_cs_v4u(dst, o[0], o[1], o[2], o[3]);
        } else {
            // edge chunk: per cell, walking Eq. 1 across the row end
            uint32_t o[4] = {0, 0, 0, 0};
            int64_t ii = i, jj = j0;
#pragma unroll 1
            for (int q = 0; q < 16; ++q) {
                while (jj > ii) { jj -= ii + 1; ++ii; }
                if (c + q < a.out_cells) o[q >> 2] |= life_cell(a, ii, jj) << (8 * (q & 3));
                ++jj;
            }
            if (c + 16 <= a.out_cells) {
                st_cs_v4u(dst, o[0], o[1], o[2], o[3]);
            } else {
#pragma unroll 1
                for (int q = 0; q < 16; ++q)
                    if (c + q < a.out_cells) dst[q] = (uint8_t)(o[q >> 2] >> (8 * (q & 3)));
            }
        }
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
