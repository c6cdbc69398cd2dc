// ca.cu -- Life B3/S23 on the triangular domain {(i, j): 0 <= j <= i < n}
// (P:79-80 names cellular automata on triangular domains, citing Conway's
// Life; cells outside the triangle are dead -- DESIGN.md reading Q11).
// State: u8 {0,1} in the packed Eq. 1 layout.  Four kernels:
//   rho = 240: multi::ca_packed_kernel -- tri_ca_run (the bench's N = 1 path): the
//              state converted once to BITS in the packed Eq. 1 order (bit T(i) + j),
//              8 generations per launch on a register-resident bitmap, converted back
//              at the end (8x less HBM traffic per launch than the byte state);
//   rho = 128, 224: multi::ca_multi_kernel -- k generations per launch on a
//              register-resident bitmap (tri_ca_steps; tri_ca_step is k = 1;
//              tri_ca_steps_p2p also stores the halo rows into peer memory);
//   rho = 256: bits::ca_bits_kernel -- one generation, shared-memory bitmaps;
//   rho = 512: ca_kernel -- one generation, byte SWAR (described next).
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
    const uint8_t *above, *below;  // halo rows [R0-k, R0) and [R1, R1+k), packed (NULL = dead)
    int64_t n, R0, R1;             // this slice owns rows [R0, R1)
    int64_t k;                     // halo depth (generations per launch)
    uint64_t base;                 // T(R0)
    uint64_t above_base;           // T(max(R0 - k, 0)): packed start of the above block
    uint64_t out_cells;
    uint64_t omega_begin, omega_end;
    int64_t tile_row_begin;
    // fused halo exchange (tri_ca_steps_p2p; NULL otherwise): rows [R0, R0 + k) are
    // also stored to peer_above + (slice offset), rows [R1 - k, R1) to peer_below +
    // (slice offset) -- the neighbours' halo buffers, mapped over NVLink
    uint8_t *peer_above, *peer_below;
};

#ifndef TRI_CA_PACKED_EXCH
#define TRI_CA_PACKED_EXCH 1
#endif
// tri_ca_run's bit-packed state: cell (i, j) at bit T(i) + j of the word array.
struct PackedArgs {
    const uint32_t *in;
    uint32_t *out;
    int64_t n, k, nwords;
    uint64_t omega_begin, omega_end;
};

// Row pointer to column 0 of row r, or nullptr for a dead row.
__device__ __forceinline__ const uint8_t *row_ptr(const CaArgs &a, int64_t r) {
    if (r < 0 || r >= a.n) return nullptr;
    if (r < a.R0) return (r >= a.R0 - a.k && a.above) ? a.above + (tri::T2((uint64_t)r) - a.above_base) : nullptr;
    if (r >= a.R1)
        return (r < a.R1 + a.k && a.below) ? a.below + (tri::T2((uint64_t)r) - tri::T2((uint64_t)a.R1)) : nullptr;
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

// Interior window: the 18 bytes at w (all inside one row of the slice buffer)
// from two aligned 16-byte loads (a third 4-byte load when the window starts at
// byte 15 of its chunk); the realignment offset is uniform across a row group.
__device__ __forceinline__ void window128(const uint8_t *w, uint32_t (&X)[5]) {
    const uintptr_t A = (uintptr_t)w;
    const uint4 *q = (const uint4 *)(A & ~(uintptr_t)15);
    const uint32_t o = (uint32_t)(A & 15u);
    const uint4 c0 = __ldg(q), c1 = __ldg(q + 1);
    const uint32_t R8 = (o == 15u) ? __ldg((const uint32_t *)(q + 2)) : 0u;
    const uint32_t R[9] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w, R8};
    const uint32_t sh = 8u * (o & 3u);
    switch (o >> 2) {
        case 0:
#pragma unroll
            for (int t = 0; t < 5; ++t) X[t] = __funnelshift_r(R[t], R[t + 1], sh);
            break;
        case 1:
#pragma unroll
            for (int t = 0; t < 5; ++t) X[t] = __funnelshift_r(R[t + 1], R[t + 2], sh);
            break;
        case 2:
#pragma unroll
            for (int t = 0; t < 5; ++t) X[t] = __funnelshift_r(R[t + 2], R[t + 3], sh);
            break;
        default:
#pragma unroll
            for (int t = 0; t < 5; ++t) X[t] = __funnelshift_r(R[t + 3], R[t + 4], sh);
            break;
    }
}

// B3/S23 on 4 cells: with nb = sum9 - self (bytes 0..8),
// alive' = (nb == 3) | (self & nb == 2)  <=>  (nb | self) == 3.
// y = (nb | self) ^ 3 has bytes <= 15, so y + 0x7f never carries between bytes
// and its bit 7 is clear exactly when y == 0.
__device__ __forceinline__ uint32_t life_word(uint32_t sum9, uint32_t self) {
    const uint32_t y = ((sum9 - self) | self) ^ 0x03030303u;
    return (~(y + 0x7f7f7f7fu) >> 7) & 0x01010101u;
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

// Interior chunk: rows given by their column-0 pointers (all in the slice).
__device__ __forceinline__ void eval16_fast(const uint8_t *pu, const uint8_t *pm, const uint8_t *pd, int64_t js,
                                            uint32_t (&o)[4]) {
    uint32_t U[5], M[5], D[5], V[5];
    window128(pu + js - 1, U);
    window128(pm + js - 1, M);
    window128(pd + js - 1, D);
#pragma unroll
    for (int t = 0; t < 5; ++t) V[t] = U[t] + M[t] + D[t];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const uint32_t sum9 = V[w] + __funnelshift_r(V[w], V[w + 1], 8) + __funnelshift_r(V[w], V[w + 1], 16);
        o[w] = life_word(sum9, __funnelshift_r(M[w], M[w + 1], 8));
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

// Raw (unaligned) 18-byte window: loads issued now, realigned later, so that a
// lane can keep the six windows of two rows in flight at once.
struct RawWin {
    uint4 c0, c1;
    uint32_t r8, o;
};

__device__ __forceinline__ RawWin load_win(const uint8_t *w) {
    const uintptr_t A = (uintptr_t)w;
    const uint4 *q = (const uint4 *)(A & ~(uintptr_t)15);
    RawWin r;
    r.o = (uint32_t)(A & 15u);
    r.c0 = __ldg(q);
    r.c1 = __ldg(q + 1);
    r.r8 = (r.o == 15u) ? __ldg((const uint32_t *)(q + 2)) : 0u;
    return r;
}

__device__ __forceinline__ void realign(const RawWin &r, uint32_t (&X)[5]) {
    const uint32_t R[9] = {r.c0.x, r.c0.y, r.c0.z, r.c0.w, r.c1.x, r.c1.y, r.c1.z, r.c1.w, r.r8};
    const uint32_t sh = 8u * (r.o & 3u);
    switch (r.o >> 2) {
        case 0:
#pragma unroll
            for (int t = 0; t < 5; ++t) X[t] = __funnelshift_r(R[t], R[t + 1], sh);
            break;
        case 1:
#pragma unroll
            for (int t = 0; t < 5; ++t) X[t] = __funnelshift_r(R[t + 1], R[t + 2], sh);
            break;
        case 2:
#pragma unroll
            for (int t = 0; t < 5; ++t) X[t] = __funnelshift_r(R[t + 2], R[t + 3], sh);
            break;
        default:
#pragma unroll
            for (int t = 0; t < 5; ++t) X[t] = __funnelshift_r(R[t + 3], R[t + 4], sh);
            break;
    }
}

__device__ __forceinline__ void life16(const RawWin &ru, const RawWin &rm, const RawWin &rd, uint32_t (&o)[4]) {
    uint32_t U[5], M[5], D[5], V[5];
    realign(ru, U);
    realign(rm, M);
    realign(rd, D);
#pragma unroll
    for (int t = 0; t < 5; ++t) V[t] = U[t] + M[t] + D[t];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const uint32_t sum9 = V[w] + __funnelshift_r(V[w], V[w + 1], 8) + __funnelshift_r(V[w], V[w + 1], 16);
        o[w] = life_word(sum9, __funnelshift_r(M[w], M[w + 1], 8));
    }
}

// Where one output chunk of row i lies (aligned-chunk ownership) and whether it
// can take the interior path.
struct ChunkPos {
    uint64_t c;          // local packed index of the chunk (16-aligned)
    int64_t i, j0;       // first cell
    const uint8_t *pm;   // column 0 of row i in the slice buffer
    bool valid, fast;
};

template <int RHO>
__device__ __forceinline__ ChunkPos chunk_pos(const CaArgs &a, int64_t i, int64_t c0, int k) {
    ChunkPos p;
    p.i = i;
    p.valid = false;
    p.fast = false;
    if (i >= a.R1 || i < a.R0) return p;
    const uint64_t s = tri::T2((uint64_t)i) + (uint64_t)c0 - a.base;   // local segment start
    const int64_t seg = i - c0 + 1;
    const int64_t len = seg < RHO ? seg : RHO;
    const int off = (int)((0u - (uint32_t)s) & 15u) + 16 * k;
    if (off >= len) return p;
    p.valid = true;
    p.c = s + (uint64_t)off;
    p.j0 = c0 + off;
    p.pm = a.in + (s - (uint64_t)c0);
    p.fast = p.j0 >= 1 && p.j0 + 16 <= i - 1 && i > a.R0 && i + 1 < a.R1;
    return p;
}

// Any chunk, including the edge cases (masked windows / row crossing / tiny rows).
__device__ __forceinline__ void chunk_general(const CaArgs &a, const ChunkPos &p) {
    const int64_t i = p.i, j0 = p.j0;
    const uint64_t c = p.c;
    uint32_t o[4];
    if (p.fast) {
        life16(load_win(p.pm - i + j0 - 1), load_win(p.pm + j0 - 1), load_win(p.pm + i + 1 + j0 - 1), o);
    } else if (j0 + 15 <= i) {
        eval16<true>(a, i, j0, o);            // touches column -1 / the diagonal / the slice edge
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
    // two rows per lane per iteration: all twelve 16-byte loads in flight together
#pragma unroll 1
    for (int rr = rs; rr < ROWS_PER_WARP; rr += 2 * RPW) {
        const ChunkPos p = chunk_pos<RHO>(a, rbase + rr, c0, k);
        const ChunkPos q = (rr + RPW < ROWS_PER_WARP) ? chunk_pos<RHO>(a, rbase + rr + RPW, c0, k) : ChunkPos{};
        const bool q_ok = rr + RPW < ROWS_PER_WARP && q.valid;
        if (p.valid && p.fast && q_ok && q.fast) {
            const RawWin pu = load_win(p.pm - p.i + p.j0 - 1), pm = load_win(p.pm + p.j0 - 1),
                         pd = load_win(p.pm + p.i + 1 + p.j0 - 1);
            const RawWin qu = load_win(q.pm - q.i + q.j0 - 1), qm = load_win(q.pm + q.j0 - 1),
                         qd = load_win(q.pm + q.i + 1 + q.j0 - 1);
            uint32_t o[4];
            life16(pu, pm, pd, o);
            store_chunk(a, p.c, o);
            life16(qu, qm, qd, o);
            store_chunk(a, q.c, o);
        } else {
            if (p.valid) chunk_general(a, p);
            if (q_ok) chunk_general(a, q);
        }
    }
}

// ============================================================================
// Bit-sliced tile (rho = 256): the CTA turns its (rho+2)-row halo tile into
// column-aligned bitmaps in shared memory (bit x of row y <-> column c0-1+x),
// evaluates B3/S23 32 cells per LOP3 chain, and expands the result to the
// aligned 16-byte output chunks it owns.  ~3 instructions per cell instead of
// ~16 for byte SWAR, which made the kernel ALU-bound.
namespace bits {

template <int RHO>
struct Cfg {
    static constexpr int NIN = RHO + 2;                 // input rows r0-1 .. r0+RHO
    static constexpr int NW = (RHO + 18 + 31) / 32;     // bitmap words per row (cols c0-1 .. c0+RHO+16)
    static constexpr int NBAND = 32;                    // phase B: NW words x 32 row bands
    static constexpr int NT = NW * NBAND;               // threads (>= NIN: one input row each in phase A)
    static_assert(NT >= NIN, "phase A needs one thread per input row");
    static_assert(RHO % NBAND == 0, "bands of whole rows");
};

// Bytes in {0,1} -> bits (byte q -> bit q).  For two words x, y of such bytes,
// u = x + 16 y holds x's byte k in bit 8k and y's in bit 8k + 4; u * 0x01020408
// moves them to bits 24 + k and 28 + k, and no two partial products share a bit
// below 32 (no carries), so byte 3 of the product = x's 4 bits | y's 4 bits << 4.
__device__ __forceinline__ uint32_t pack_pair(uint32_t x, uint32_t y) { return (y * 16u + x) * 0x01020408u; }
// 16 bytes -> 16 bits
__device__ __forceinline__ uint32_t pack16(const uint4 c) {
    return __byte_perm(pack_pair(c.x, c.y), pack_pair(c.z, c.w), 0x7373) & 0xffffu;
}
// 32 bytes (lo: columns 0-15, hi: 16-31) -> 32 bits
__device__ __forceinline__ uint32_t pack32(const uint4 lo, const uint4 hi) {
    const uint32_t a = __byte_perm(pack_pair(lo.x, lo.y), pack_pair(lo.z, lo.w), 0x7373);
    const uint32_t b = __byte_perm(pack_pair(hi.x, hi.y), pack_pair(hi.z, hi.w), 0x7373);
    return __byte_perm(a, b, 0x5410);
}

// 4 bits -> 4 bytes {0,1}: nibble * 0x00204081 puts bit q at 8q (no collisions).
__device__ __forceinline__ uint32_t spread4(uint32_t v) { return (v * 0x00204081u) & 0x01010101u; }

// One LOP3 with truth table F over (a, b, c) = (0xf0, 0xcc, 0xaa).
template <int F>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(F));
    return d;
}
// Integer multiply-adds (FMA pipe): lo(a b) + c and hi(a b) + c.
__device__ __forceinline__ uint32_t imad_lo(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t imad_hi(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

template <int RHO>
struct Smem {
    uint32_t in[Cfg<RHO>::NIN][Cfg<RHO>::NW];
    uint32_t out[RHO][Cfg<RHO>::NW];
};

// Byte mask of chunk bytes [lo, hi) (clamped to the 16-byte chunk) applied in place.
__device__ __forceinline__ uint32_t word_mask(int64_t lo_c, int64_t hi_c, int u) {
    const int lo = (int)(lo_c - 4 * u), hi = (int)(hi_c - 4 * u);
    const int l = lo < 0 ? 0 : (lo > 4 ? 4 : lo), g = hi < 0 ? 0 : (hi > 4 ? 4 : hi);
    return g <= l ? 0u : ((0xffffffffu >> (8 * (4 - g))) & (0xffffffffu << (8 * l)));
}
__device__ __forceinline__ void mask_chunk(uint4 &c, int64_t lo_c, int64_t hi_c) {
    c.x &= word_mask(lo_c, hi_c, 0);
    c.y &= word_mask(lo_c, hi_c, 1);
    c.z &= word_mask(lo_c, hi_c, 2);
    c.w &= word_mask(lo_c, hi_c, 3);
}

template <int RHO>
__device__ __forceinline__ void phase_a_row(const CaArgs &a, int64_t r, int64_t c0, uint32_t *dst) {
    constexpr int NW = Cfg<RHO>::NW;
    const uint8_t *p = row_ptr(a, r);
    if (!p) {
#pragma unroll
        for (int w = 0; w < NW; ++w) dst[w] = 0;
        return;
    }
    const int64_t cs = c0 - 1;                            // column of bitmap bit 0
    const uintptr_t A = (uintptr_t)(p + cs);
    const uint4 *q = (const uint4 *)(A & ~(uintptr_t)15);
    const uint32_t e = (uint32_t)(A & 15u);
    const int64_t col0 = cs - (int64_t)e;                 // column of chunk 0's byte 0
    // every loaded byte inside [0, r]: no masks, no out-of-row loads
    const bool full = col0 >= 0 && col0 + 32 * (NW + 1) - 1 <= r;
    uint32_t prev = 0;
#pragma unroll
    for (int v = 0; v <= NW; ++v) {
        uint32_t lo, hi;
        if (full) {
            lo = pack16(__ldg(q + 2 * v));
            hi = pack16(__ldg(q + 2 * v + 1));
        } else {
            uint32_t m2[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t cb = col0 + 32 * v + 16 * h;           // column of this chunk's byte 0
                const int64_t lo_c = cb < 0 ? -cb : 0;
                const int64_t hi_c = r - cb + 1;                      // valid bytes [lo_c, hi_c)
                if (lo_c >= 16 || hi_c <= 0 || lo_c >= hi_c) {
                    m2[h] = 0;
                } else {
                    // zero the bytes outside [lo_c, hi_c) BEFORE packing: pack16's multiply
                    // is only collision-free for bytes in {0,1}, and bytes beyond the row
                    // (or the buffer) may hold anything
                    uint4 c = __ldg(q + 2 * v + h);
                    uint32_t *cw = &c.x;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int lo = (int)(lo_c - 4 * u), hi = (int)(hi_c - 4 * u);
                        const int l = lo < 0 ? 0 : (lo > 4 ? 4 : lo), g = hi < 0 ? 0 : (hi > 4 ? 4 : hi);
                        const uint32_t mk = g <= l ? 0u : ((0xffffffffu >> (8 * (4 - g))) & (0xffffffffu << (8 * l)));
                        cw[u] &= mk;
                    }
                    m2[h] = pack16(c);
                }
            }
            lo = m2[0];
            hi = m2[1];
        }
        const uint32_t P = lo | (hi << 16);               // stream bits [32v - e, 32v - e + 32)
        if (v > 0) dst[v - 1] = __funnelshift_r(prev, P, e);
        prev = P;
    }
}

template <int RHO>
__device__ __forceinline__ void tile(const CaArgs &a, uint32_t bi, uint32_t bj, Smem<RHO> &sm) {
    constexpr int NIN = Cfg<RHO>::NIN, NW = Cfg<RHO>::NW, NT = Cfg<RHO>::NT, NBAND = Cfg<RHO>::NBAND;
    const int t = threadIdx.x;
    const int64_t r0 = (int64_t)bi * RHO, c0 = (int64_t)bj * RHO;
    // ---- A: rows r0-1 .. r0+RHO -> bitmaps (one row per thread)
    if (t < NIN) phase_a_row<RHO>(a, r0 - 1 + t, c0, sm.in[t]);
    __syncthreads();
    // ---- B: B3/S23 on words; thread = (word w, band of 8 output rows)
    {
        const int w = t % NW, band = t / NW;
        constexpr int ROWS = RHO / NBAND;
        const int y0 = band * ROWS;                       // first output row (in-row y0 + 1)
        uint32_t h0u, h1u, p0m, p1m, Wm;                  // rolling: up row sums, mid pair sums
        auto row_terms = [&](int yin, uint32_t &h0, uint32_t &h1, uint32_t &p0, uint32_t &p1, uint32_t &W) {
            W = sm.in[yin][w];
            const uint32_t Wp = w > 0 ? sm.in[yin][w - 1] : 0u;
            const uint32_t Wn = w + 1 < NW ? sm.in[yin][w + 1] : 0u;
            const uint32_t L = __funnelshift_l(Wp, W, 1);   // left neighbour of bit b = bit b-1
            const uint32_t R = __funnelshift_r(W, Wn, 1);   // right neighbour
            h0 = L ^ W ^ R;
            h1 = (L & W) | (L & R) | (W & R);
            p0 = L ^ R;
            p1 = L & R;
        };
        uint32_t d0, d1, dp0, dp1, dW;
        row_terms(y0, h0u, h1u, p0m, p1m, Wm);            // row above the band
        uint32_t tmp0, tmp1;
        row_terms(y0 + 1, tmp0, tmp1, p0m, p1m, Wm);      // first mid row
        uint32_t h0m = tmp0, h1m = tmp1;
#pragma unroll 1
        for (int y = 0; y < ROWS; ++y) {
            row_terms(y0 + y + 2, d0, d1, dp0, dp1, dW);  // row below
            // nb = (h0u + 2 h1u) + (h0d + 2 h1d) + (p0m + 2 p1m); alive' <=> (nb | self) == 3
            const uint32_t z0 = h0u ^ d0 ^ p0m;
            const uint32_t k0 = (h0u & d0) | (h0u & p0m) | (d0 & p0m);
            const uint32_t x = h1u ^ d1 ^ p1m;
            const uint32_t ge2 = (h1u & d1) | (h1u & p1m) | (d1 & p1m);
            const uint32_t one = ~ge2 & (x ^ k0);             // exactly one of {h1u, h1d, p1m, k0}
            sm.out[y0 + y][w] = one & (z0 | Wm);
            h0u = h0m; h1u = h1m;                             // mid becomes up
            h0m = d0; h1m = d1; p0m = dp0; p1m = dp1; Wm = dW;
        }
    }
    __syncthreads();
    // ---- C: expand + aligned 16-byte stores; thread = (row, chunk slot)
    constexpr int L = RHO / 16;                           // chunk slots per row
#pragma unroll 1
    for (int idx = t; idx < RHO * L; idx += NT) {
        const int rr = idx / L, k = idx % L;
        const int64_t i = r0 + rr;
        if (i >= a.R1 || i < a.R0) continue;
        const uint64_t s = tri::T2((uint64_t)i) + (uint64_t)c0 - a.base;
        const int64_t seg = i - c0 + 1;
        const int64_t len = seg < RHO ? seg : RHO;
        const int off = (int)((0u - (uint32_t)s) & 15u) + 16 * k;
        if (off >= len) continue;
        const int64_t j0 = c0 + off;
        if (j0 + 15 > i) {                                    // crosses the row end: SWAR edge path
            ChunkPos p;
            p.i = i; p.j0 = j0; p.c = s + (uint64_t)off; p.pm = nullptr; p.valid = true; p.fast = false;
            chunk_general(a, p);
            continue;
        }
        const int x = off + 1;                                // bitmap bit of column j0
        const uint32_t w0 = sm.out[rr][x >> 5];
        const uint32_t w1 = (x >> 5) + 1 < NW ? sm.out[rr][(x >> 5) + 1] : 0u;
        const uint32_t b = __funnelshift_r(w0, w1, (uint32_t)(x & 31));
        st_cs_v4u(a.out + s + (uint64_t)off, spread4(b & 15u), spread4((b >> 4) & 15u), spread4((b >> 8) & 15u),
                  spread4((b >> 12) & 15u));
    }
}

template <int RHO, int STRAT>
__global__ void __launch_bounds__(Cfg<RHO>::NT) ca_bits_kernel(CaArgs a) {
    __shared__ __align__(16) Smem<RHO> sm;
    if (STRAT == TRI_BB) {
        const uint32_t bj = blockIdx.x;
        const uint32_t bi = blockIdx.y + (uint32_t)a.tile_row_begin;
        if (bj > bi) return;
    }
    if (STRAT == TRI_BB) {
        tile<RHO>(a, blockIdx.y + (uint32_t)a.tile_row_begin, blockIdx.x, sm);
    } else if (STRAT == TRI_LAMBDA) {
        const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (w >= a.omega_end) return;
        uint32_t bi, bj;
        tri::lambda_map(w, bi, bj);
        tile<RHO>(a, bi, bj, sm);
    } else {
#pragma unroll 1
        for (tri::TileWalk t(a.omega_begin, a.omega_end); t.more(); t.next()) {
            tile<RHO>(a, t.bi, t.bj, sm);
            __syncthreads();                                  // smem reused by the next tile
        }
    }
}

template <int RHO>
tri_status launch(const tri_map_t &m, int strategy, CaArgs a, cudaStream_t st) {
    constexpr int NT = Cfg<RHO>::NT;
    if (strategy == TRI_BB) {
        const int64_t tr0 = m.row_begin / m.rho;
        const int64_t tr1 = (m.row_end + m.rho - 1) / m.rho;
        if (tr1 <= tr0) return TRI_OK;
        if (tr1 - tr0 > 65535) return TRI_ENOTSUP;
        a.tile_row_begin = tr0;
        ca_bits_kernel<RHO, TRI_BB><<<dim3((unsigned)m.m, (unsigned)(tr1 - tr0)), NT, 0, st>>>(a);
    } else if (strategy == TRI_LAMBDA) {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        ca_bits_kernel<RHO, TRI_LAMBDA><<<tri::tile_grid(nb), NT, 0, st>>>(a);
    } else {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ca_bits_kernel<RHO, TRI_LAMBDA_PERSIST>, NT, 0);
        uint64_t g = (uint64_t)tri::sm_count() * (uint64_t)(per_sm > 0 ? per_sm : 1);
        if (g > nb) g = nb;
        ca_bits_kernel<RHO, TRI_LAMBDA_PERSIST><<<(unsigned)g, NT, 0, st>>>(a);
    }
    tri::note_launches(1);
    return tri::cuda_status();
}

}  // namespace bits

// ============================================================================
// k generations per launch (temporal blocking with deep halos);
// also tri_ca_step at rho = 128 / 224 (k = 1).  rho x rho tiles; the CTA loads rows
// [r0-k, r0+rho+k) x columns [c0-k, c0+rho+k), packs them to bitmaps, runs k
// generations with the bitmap in registers -- re-masking the triangle after
// each one -- and writes only its own row segments [c0, min(c0+rho, i+1)): aligned chunks
// with 16-byte streaming stores, the partial chunks at segment ends byte-wise
// (a neighbouring tile writes the other bytes of such a chunk).  Garbage from
// the region edge moves one cell per generation, so after k generations the
// central rho x rho block is exact.  HBM traffic per cell-generation falls from
// 2 bytes to about (1.2 + 1) / k bytes.
namespace multi {

constexpr int RB = 4;                    // phase B: rows per band (register-resident)

template <bool B> struct MaskTag { static constexpr bool value = B; };

// bits of columns [cb, cb + 32) that lie inside row r of the triangle
__device__ __forceinline__ uint32_t tri_mask(int64_t r, int64_t n, int64_t cb) {
    if (r < 0 || r >= n) return 0u;
    const int64_t lo = cb < 0 ? -cb : 0;              // first valid bit
    const int64_t hi = r - cb + 1;                    // one past the last valid bit
    if (hi <= 0 || lo >= 32 || lo >= hi) return 0u;
    const uint32_t up = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
    return up & ~((1u << lo) - 1u);
}

// Geometry: rho x rho tiles, NW bitmap words per region row (bit x <-> column
// c0 - k + x), WPT horizontally adjacent words per phase-B thread, k <= KMAX.
//   <128, 5, 1,  8>: 160 columns, 192 threads (rho = 128, k <= 8)
//   <128, 6, 1, 16>: 192 columns, 256 threads (rho = 128, k <= 16)
//   <224, 8, 2,  8>: 256 columns, 256 threads (rho = 224, k <= 8): the region
//       overhead (32 NW)(rho + 2k) / rho^2 falls from 1.41 to 1.22 at k = 8, no
//       phase-B lane idles (4 threads per band, 8 bands per warp), and the word
//       pair a thread owns halves the shuffles per cell (the inner neighbour bits
//       come from the thread's own other word).
template <int RHO_, int NWV, int WPT_, int KMAX_, int SPILL_ = 15>
struct Multi {
    static constexpr int RHO = RHO_;
    static constexpr int NW = NWV;
    static constexpr int WPT = WPT_;
    static constexpr int KMAX = KMAX_;
    // garbage from the right edge reaches column c0 + 32 NW - 2K; the byte store phase reads
    // up to c0 + rho + 14 (SPILL = 15), the bit-packed one up to c0 + rho - 1 (SPILL = 0)
    static_assert(32 * NW - 2 * KMAX >= RHO + SPILL_, "bitmap too narrow for KMAX");
    static_assert(NW % WPT == 0 && RHO % 16 == 0, "geometry");
    static constexpr int NINMAX = RHO + 2 * KMAX;          // region rows
    static constexpr int TPB = NW / WPT;                   // threads per band
    static constexpr int BPW = 32 / TPB;                   // bands per warp (lanes past BPW TPB idle in B)
    static constexpr int NBAND = NINMAX / RB;
    static constexpr int NT = 32 * ((NBAND + BPW - 1) / BPW);
    static_assert(NBAND * RB == NINMAX, "bands tile the region");
    static_assert(NT >= NINMAX, "phase A: one thread per region row");
    static constexpr int RAWB = 32 * (NW + 1);             // loaded bytes per row (>= 15 + rho + 2k)
    static constexpr int NCH = RAWB / 16;
    // phase C: LPR lanes per row, CPL consecutive 16-byte chunks per lane (two
    // chunks per lane measured faster at rho = 224, slower at rho = 128 / k = 1)
    static constexpr int LPR = 8;
    static constexpr int CPL = RHO <= 128 ? 1 : 2;
    static_assert(16 * CPL * LPR >= RHO && NT % LPR == 0, "phase C slots");

    static constexpr int AW = NW | 1;                      // odd row stride: phase A's row-per-lane stores conflict-free
    struct Smem {
        uint32_t A[NINMAX][AW];                            // packed region (phase A) / final state (phase C)
        uint2 top[2][NBAND][NW], bot[2][NBAND][NW];        // band edge row sums (s0, s1), double-buffered
        uint64_t seg[RHO];
    };

// ---- B (shared by the byte and the bit-packed tile forms): K generations on the region
// bitmap sm.A (rows r0 - K .., bit x <-> column cs + x); the result is left in sm.A.
template <bool EXCH>
static __device__ __forceinline__ void phase_b(const int64_t n, const int K, const int NIN, const int64_t r0,
                                               const int64_t cs, Smem &sm) {
    const int t = threadIdx.x;
    struct { int64_t n; } a{n};
    // K generations with the state in registers.  Thread (band, w) owns
    // bitmap word w of region rows [RB band, RB band + RB); horizontal neighbour
    // words come by shuffle (lane +-1), the rows above / below the band through
    // shared memory (one exchange per generation).  What enters at the region
    // edges (the shuffle partners of words 0 and NW-1, rows past the staged
    // region, idle lanes) is garbage that moves one cell per generation: after K
    // generations it reaches column c0 - 1 on the left, c0 + 32 NW - 2K >= c0 + rho
    // + 15 on the right and rows outside [K, K + rho) -- never a cell phase C writes.
    // Cells outside the triangle are re-masked dead every generation (skipped
    // when the whole CTA's mask is all ones).
    {
        const int lane = t & 31;
        const bool act = lane < BPW * TPB;
        const int w0 = act ? (lane % TPB) * WPT : 0;         // first owned word
        const int band = (t >> 5) * BPW + (act ? lane / TPB : 0);
        const bool live = act && band < NBAND;
        uint32_t X[RB][WPT], Mk[RB][WPT];
        // CTA-uniform: every region cell (rows r0-K .. r0+rho+K-1, bitmap columns
        // cs .. cs+32 NW-1) inside the triangle and the domain -> no masks at all
        const bool inside = cs >= 0 && cs + 32 * NW - 1 <= r0 - K && r0 + RHO + K <= a.n;
        bool ones = true;
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            const int y = RB * band + q;
            const bool in = live && y < NIN;
#pragma unroll
            for (int u = 0; u < WPT; ++u) {
                X[q][u] = in ? sm.A[y][w0 + u] : 0u;
                Mk[q][u] = (in && !inside) ? tri_mask(r0 - K + y, a.n, cs + 32 * (w0 + u)) : 0xffffffffu;
                ones = ones && Mk[q][u] == 0xffffffffu;
            }
        }
        // block-uniform (the generation loops below contain __syncthreads)
        const bool nomask = __syncthreads_and(inside || ones) != 0;
        // The ALU pipe (LOP3 / SHF) and the shuffle path are the limiters of phase B;
        // the FMA pipe runs at the ALU's rate beside it, so the one-bit neighbour
        // shifts go there as integer multiply-adds (L = 2V + (left >> 31),
        // R = hi(V 2^31) + (right << 31)), and the logic is written as explicit
        // 3-input LOP3s (the compiler's own factoring took 61 instead of 44 per
        // 4 x 32 cells).  The multipliers 2 and 2^31 are hidden from the compiler
        // (it would turn the multiply-adds back into ALU-pipe LEA.HI / SHF); a.n < 2^62.
        const uint32_t two = 2u | (uint32_t)((uint64_t)a.n >> 62);
        const uint32_t half = two << 30;
        // row sums of one region row: s = L + V + R (bits s0, s1), p = L + R (p0, p1)
        auto hsum = [&](const uint32_t (&V)[WPT], uint32_t (&s0)[WPT], uint32_t (&s1)[WPT], uint32_t (&q0)[WPT],
                        uint32_t (&q1)[WPT], bool need_q) {
            const uint32_t Vp = __shfl_up_sync(0xffffffffu, V[WPT - 1], 1);   // left thread's last word
            const uint32_t Vn = __shfl_down_sync(0xffffffffu, V[0], 1);       // right thread's first word
#pragma unroll
            for (int u = 0; u < WPT; ++u) {
                const uint32_t lw = u == 0 ? Vp : V[u - 1], rw = u == WPT - 1 ? Vn : V[u + 1];
                const uint32_t L = bits::imad_lo(V[u], two, bits::imad_hi(lw, two, 0u));
                const uint32_t R = bits::imad_hi(V[u], half, bits::imad_lo(rw, half, 0u));
                s0[u] = bits::lop3<0x96>(L, V[u], R);
                s1[u] = bits::lop3<0xe8>(L, V[u], R);
                if (need_q) {
                    q0[u] = L ^ R;
                    q1[u] = L & R;
                }
            }
        };
        auto generations = [&](auto masked) {
#pragma unroll 1
            for (int g = 0; g < K; ++g) {
                const int pb = g & 1;
                uint32_t h0[RB + 2][WPT], h1[RB + 2][WPT], p0[RB][WPT], p1[RB][WPT];
                if constexpr (EXCH) {
                    // own rows' sums first; the band's first / last row sums go to the
                    // neighbouring bands (which would otherwise recompute them: 2 of every
                    // RB + 2 row sums)
#pragma unroll
                    for (int q = 0; q < RB; ++q) hsum(X[q], h0[q + 1], h1[q + 1], p0[q], p1[q], true);
                    if (live) {
#pragma unroll
                        for (int u = 0; u < WPT; ++u) {
                            sm.top[pb][band][w0 + u] = make_uint2(h0[1][u], h1[1][u]);
                            sm.bot[pb][band][w0 + u] = make_uint2(h0[RB][u], h1[RB][u]);
                        }
                    }
                    __syncthreads();
#pragma unroll
                    for (int u = 0; u < WPT; ++u) {
                        const uint2 up = (live && band > 0) ? sm.bot[pb][band - 1][w0 + u] : make_uint2(0u, 0u);
                        const uint2 dn =
                            (live && band + 1 < NBAND) ? sm.top[pb][band + 1][w0 + u] : make_uint2(0u, 0u);
                        h0[0][u] = up.x; h1[0][u] = up.y;
                        h0[RB + 1][u] = dn.x; h1[RB + 1][u] = dn.y;
                    }
                } else {
                    // the band's edge rows go to the neighbouring bands, which form their sums
                    if (live) {
#pragma unroll
                        for (int u = 0; u < WPT; ++u) {
                            sm.top[pb][band][w0 + u].x = X[0][u];
                            sm.bot[pb][band][w0 + u].x = X[RB - 1][u];
                        }
                    }
                    __syncthreads();
                    uint32_t up[WPT], dn[WPT], u0[WPT], u1[WPT];
#pragma unroll
                    for (int u = 0; u < WPT; ++u) {
                        up[u] = (live && band > 0) ? sm.bot[pb][band - 1][w0 + u].x : 0u;
                        dn[u] = (live && band + 1 < NBAND) ? sm.top[pb][band + 1][w0 + u].x : 0u;
                    }
                    hsum(up, h0[0], h1[0], u0, u1, false);
#pragma unroll
                    for (int q = 0; q < RB; ++q) hsum(X[q], h0[q + 1], h1[q + 1], p0[q], p1[q], true);
                    hsum(dn, h0[RB + 1], h1[RB + 1], u0, u1, false);
                }
#pragma unroll
                for (int q = 0; q < RB; ++q) {
#pragma unroll
                    for (int u = 0; u < WPT; ++u) {
                        // neighbour count = h(row above) + h(row below) + p(own row), bit-sliced:
                        // count = z0 + 2 (x + k0) + 4 ge2; alive' <=> count == 3, or count == 2
                        // and alive <=> (x + k0 + 2 ge2 == 1) and (z0 | alive)
                        const uint32_t a0 = h0[q][u], b0 = h0[q + 2][u], c0_ = p0[q][u];
                        const uint32_t a1 = h1[q][u], b1 = h1[q + 2][u], c1 = p1[q][u];
                        const uint32_t z0 = bits::lop3<0x96>(a0, b0, c0_);
                        const uint32_t k0 = bits::lop3<0xe8>(a0, b0, c0_);
                        const uint32_t x = bits::lop3<0x96>(a1, b1, c1);
                        const uint32_t ge2 = bits::lop3<0xe8>(a1, b1, c1);
                        const uint32_t one = bits::lop3<0x06>(ge2, x, k0);      // ~ge2 & (x ^ k0)
                        const uint32_t nx = bits::lop3<0xe0>(one, z0, X[q][u]); // one & (z0 | X)
                        X[q][u] = decltype(masked)::value ? nx & Mk[q][u] : nx;
                    }
                }
            }
        };
        if (nomask) generations(MaskTag<false>{});
        else generations(MaskTag<true>{});
        __syncthreads();                                      // last exchange read before A is overwritten
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            const int y = RB * band + q;
#pragma unroll
            for (int u = 0; u < WPT; ++u)
                if (live && y < NINMAX) sm.A[y][w0 + u] = X[q][u];
        }
        __syncthreads();
    }
}

// P2P: the slice's first / last k rows also go to the neighbours' halo buffers (peer
// memory); a compile-time flag so the plain launch carries none of that logic.
template <bool P2P>
static __device__ __forceinline__ void tile(const CaArgs &a, uint32_t bi, uint32_t bj, Smem &sm) {
    const int t = threadIdx.x;
    const int K = (int)a.k;
    const int NIN = RHO + 2 * K;
    const int64_t r0 = (int64_t)bi * RHO, c0 = (int64_t)bj * RHO;
    const int64_t cs = c0 - K;                        // column of bitmap bit 0
    // ---- A: load + pack rows r0-K .. r0+RHO+K-1 (thread t = input row t): the
    // row's 16-byte-aligned window straight into registers (read-only path),
    // bytes outside the row masked before packing.  (Per-row cp.async.bulk
    // copies serialise on the uniform datapath -- one ELECT/R2UR round per lane
    // -- which made staging 40 % of the tile time.)
    if (t < NIN) {
        const int64_t r = r0 - K + t;
        if (t >= K && t < K + RHO) sm.seg[t - K] = tri::T2((uint64_t)r) + (uint64_t)c0 - a.base;
        const uint8_t *p = row_ptr(a, r);
        if (!p) {
#pragma unroll
            for (int v = 0; v < NW; ++v) sm.A[t][v] = 0u;
        } else {
            const uintptr_t Ad = (uintptr_t)(p + cs);
            const uint32_t e = (uint32_t)(Ad & 15u);
            const int64_t col0 = cs - (int64_t)e;
            const uint4 *q = (const uint4 *)(Ad & ~(uintptr_t)15);
            if (col0 >= 0 && col0 + RAWB - 1 <= r) {
                // whole window inside the row (hence inside the triangle): no masks
                uint4 c[NCH];
#pragma unroll
                for (int h = 0; h < NCH; ++h) c[h] = __ldg(q + h);
                uint32_t prev = bits::pack32(c[0], c[1]);
#pragma unroll
                for (int v = 1; v <= NW; ++v) {
                    const uint32_t P = bits::pack32(c[2 * v], c[2 * v + 1]);
                    sm.A[t][v - 1] = __funnelshift_r(prev, P, e);
                    prev = P;
                }
            } else {
                uint4 c[NCH];
#pragma unroll
                for (int h = 0; h < NCH; ++h) {
                    const int64_t cb = col0 + 16 * h;
                    const int64_t lo_c = cb < 0 ? -cb : 0, hi_c = r - cb + 1;
                    c[h] = make_uint4(0, 0, 0, 0);
                    if (lo_c < 16 && hi_c > 0 && lo_c < hi_c) {
                        c[h] = __ldg(q + h);
                        bits::mask_chunk(c[h], lo_c, hi_c);
                    }
                }
                uint32_t prev = 0;
#pragma unroll
                for (int v = 0; v <= NW; ++v) {
                    const uint32_t P = bits::pack32(c[2 * v], c[2 * v + 1]);
                    if (v > 0)
                        sm.A[t][v - 1] = __funnelshift_r(prev, P, e) & tri_mask(r, a.n, cs + 32 * (v - 1));
                    prev = P;
                }
            }
        }
    }
    __syncthreads();
    phase_b<false>(a.n, K, NIN, r0, cs, sm);
    uint32_t (*fin)[AW] = sm.A;
    // ---- C: aligned-chunk ownership (a 16-byte chunk is written by the tile
    // holding its first cell; the region covers the <= 15-column spill past the
    // tile for K <= KMAX).  Byte stores only where a chunk crosses a row boundary:
    // the row-i part of a chunk running past the row end (diagonal tiles), and
    // the head bytes of a row whose first chunk started in the previous row (c0 = 0).
    // LPR lanes per row, CPL consecutive chunks per lane (one 32-bit window of the
    // bitmap), 32 / LPR rows per warp pass.  A row segment of len <= rho cells
    // starting at phase delta has chunks at delta + 16 c < len, c < rho / 16.
    const int slot = t & (LPR - 1);
    // owned tile rows [rr_lo, rr_hi) and the row offset r0 - c0, in 32 bits
    const int64_t lo64 = a.R0 - r0, hi64 = a.R1 - r0;
    const int rr_lo = lo64 < 0 ? 0 : (lo64 > RHO ? RHO : (int)lo64);
    const int rr_hi = hi64 < 0 ? 0 : (hi64 > RHO ? RHO : (int)hi64);
    const int64_t dr64 = r0 - c0 + 1;                         // seg(rr) = dr + rr cells in the row from c0
    const int dr = dr64 > (1 << 20) ? (1 << 20) : (dr64 < -RHO ? -RHO : (int)dr64);
    constexpr bool p2p = P2P;
    auto chunk = [](uint32_t h) {                             // 16 bits -> 16 bytes {0,1}
        return make_uint4(bits::spread4(h & 15u), bits::spread4((h >> 4) & 15u), bits::spread4((h >> 8) & 15u),
                          bits::spread4((h >> 12) & 15u));
    };
#pragma unroll 1
    for (int rr = t / LPR + rr_lo; rr < rr_hi; rr += NT / LPR) {
        const int seg = dr + rr;
        if (seg <= 0) continue;
        const int len = seg < RHO ? seg : RHO;
        const uint64_t s = sm.seg[rr];
        const int delta = (int)((0u - (uint32_t)s) & 15u);
        const int y = rr + K;
        // this row's extra destinations: the neighbours' halo buffers (P2P), when it
        // is among the first / last k rows of the slice
        uint8_t *pa = nullptr, *pb = nullptr;
        if (p2p) {
            const int64_t r = r0 + rr;
            pa = r < a.R0 + K ? a.peer_above : nullptr;
            pb = r >= a.R1 - K ? a.peer_below : nullptr;
        }
        auto put16 = [&](uint64_t o, const uint4 v) {
            st_cs_v4u(a.out + o, v.x, v.y, v.z, v.w);
            if (pa) st_cs_v4u(pa + o, v.x, v.y, v.z, v.w);
            if (pb) st_cs_v4u(pb + o, v.x, v.y, v.z, v.w);
        };
        auto put1 = [&](uint64_t o, uint8_t v) {
            a.out[o] = v;
            if (pa) pa[o] = v;
            if (pb) pb[o] = v;
        };
        if (slot == 0 && c0 == 0) {                           // head bytes of the row (c0 = 0 only)
            const int hb = delta < len ? delta : len;
#pragma unroll 1
            for (int u = 0; u < hb; ++u) {
                const int x = u + K;
                put1(s + u, (uint8_t)((fin[y][x >> 5] >> (x & 31)) & 1u));
            }
        }
        const int off = delta + 16 * CPL * slot;              // chunks [off, off + 16) (and [off + 16, off + 32))
        if (off >= len) continue;
        const int x = off + K, wi = x >> 5;
        const uint32_t w0 = fin[y][wi];
        const uint32_t w1 = wi + 1 < NW ? fin[y][wi + 1] : 0u;
        const uint32_t b = __funnelshift_r(w0, w1, (uint32_t)(x & 31));   // cells off .. off + 31
        const uint64_t o = s + off;
        const bool second = CPL == 2 && off + 16 < len;       // a second chunk, and it is this tile's
        if (CPL == 2 && second && off + 32 <= seg) {
            put16(o, chunk(b));
            put16(o + 16, chunk(b >> 16));
        } else {
            // a chunk crossing the row end: its row-i part only (if the second chunk
            // exists and crosses, the first is full)
            const int end = seg - off < 32 ? seg - off : 32;
            int u = 0;
            if (off + 16 <= seg) {
                put16(o, chunk(b));
                u = 16;
            }
            if (u == 0 || second) {
#pragma unroll 1
                for (; u < end; ++u) put1(o + u, (uint8_t)((b >> u) & 1u));
            }
        }
    }
    // P2P: release the peer stores at system scope (NVLink): every store this thread made
    // to a neighbour's halo buffer is performed before anything the thread -- hence the
    // kernel, hence the stream's next operation (the epoch's all-reduce, whose completion
    // the neighbour's next launch waits for) -- does afterwards.
    if (P2P) __threadfence_system();
}


// ---- the bit-packed form (tri_ca_run): the state lives in HBM as packed bits, cell (i, j) at
// bit T(i) + j (32 cells per 32-bit word).  A: each region row's NW + 1 covering words, one
// funnel shift, the triangle mask; B: as above; C: the tile's row segments as whole words
// (plain stores) and at most two partial words per row (atomicOr into a zeroed buffer: a
// partial word's other bits belong to the neighbouring tile or row).
static __device__ __forceinline__ void tile_packed(const PackedArgs &a, uint32_t bi, uint32_t bj, Smem &sm) {
    const int t = threadIdx.x;
    const int K = (int)a.k;
    const int NIN = RHO + 2 * K;
    const int64_t r0 = (int64_t)bi * RHO, c0 = (int64_t)bj * RHO;
    const int64_t cs = c0 - K;                        // column of bitmap bit 0
    // CTA-uniform: every region cell inside the triangle and the domain -> no masks
    const bool inside = cs >= 0 && cs + 32 * NW - 1 <= r0 - K && r0 + RHO + K <= a.n;
    if (t < NIN) {
        const int64_t r = r0 - K + t;
        if (r < 0 || r >= a.n) {
#pragma unroll
            for (int v = 0; v < NW; ++v) sm.A[t][v] = 0u;
        } else {
            const int64_t b0 = (int64_t)tri::T2((uint64_t)r) + cs;          // bit of column cs (may be < 0)
            const int64_t w0 = b0 >= 0 ? (b0 >> 5) : -((31 - b0) >> 5);      // floor(b0 / 32)
            const uint32_t sh = (uint32_t)(b0 - 32 * w0);
            uint32_t wd[NW + 1];
            if (w0 >= 0 && w0 + NW < a.nwords) {
#pragma unroll
                for (int v = 0; v <= NW; ++v) wd[v] = __ldg(a.in + w0 + v);
            } else {
#pragma unroll
                for (int v = 0; v <= NW; ++v) {
                    const int64_t w = w0 + v;
                    wd[v] = (w >= 0 && w < a.nwords) ? __ldg(a.in + w) : 0u;
                }
            }
            if (inside) {
#pragma unroll
                for (int v = 0; v < NW; ++v) sm.A[t][v] = __funnelshift_r(wd[v], wd[v + 1], sh);
            } else {
#pragma unroll
                for (int v = 0; v < NW; ++v)
                    sm.A[t][v] = __funnelshift_r(wd[v], wd[v + 1], sh) & tri_mask(r, a.n, cs + 32 * v);
            }
        }
    }
    __syncthreads();
    phase_b<TRI_CA_PACKED_EXCH>(a.n, K, NIN, r0, cs, sm);
    uint32_t (*fin)[AW] = sm.A;
    // C: one thread per tile row: the row segment's words, whole ones by plain stores, the
    // partial first / last word by atomicOr (per-row set-up once, ~10 instructions a word)
    for (int rr = t; rr < RHO; rr += NT) {
        const int64_t r = r0 + rr;
        if (r >= a.n) break;
        const int64_t seg = r - c0 + 1;
        if (seg <= 0) continue;
        const int len = seg < RHO ? (int)seg : RHO;
        const int64_t s = (int64_t)tri::T2((uint64_t)r) + c0;           // first bit of the segment
        uint32_t *dst = a.out + (s >> 5);
        int x = (int)(32 * (s >> 5) - s) + K;                           // bitmap bit of the word's bit 0
        const uint32_t *row = fin[rr + K];
        // first word: may start before the segment (x < K) -- bits below the segment masked off
        {
            const int off = x - K;                                      // in [-31, 0]
            const uint32_t val = x >= 0 ? __funnelshift_r(row[x >> 5], row[(x >> 5) + 1], (uint32_t)(x & 31))
                                        : row[0] << (uint32_t)(-x);
            const int phi = len - off < 32 ? len - off : 32;
            const uint32_t msk = (phi >= 32 ? 0xffffffffu : ((1u << phi) - 1u)) & ~((1u << (-off)) - 1u);
            if (msk == 0xffffffffu) dst[0] = val;
            else atomicOr(dst, val & msk);
        }
        int off = x - K + 32;
        x += 32;
#pragma unroll 1
        for (int e = 1; off < len; ++e, off += 32, x += 32) {
            const int wi = x >> 5;
            const uint32_t val = __funnelshift_r(row[wi], wi + 1 < NW ? row[wi + 1] : 0u, (uint32_t)(x & 31));
            if (len - off >= 32) dst[e] = val;
            else atomicOr(dst + e, val & ((1u << (len - off)) - 1u));
        }
    }
}
};

using G5 = Multi<128, 5, 1, 8>;     // rho = 128, k <= 8
using G6 = Multi<128, 6, 1, 16>;    // rho = 128, 9 <= k <= 16
using G8 = Multi<224, 8, 2, 8>;     // rho = 224, k <= 8
using G8P = Multi<240, 8, 2, 8, 0>; // rho = 240, k <= 8, bit-packed state only: 256 columns = rho + 2k

// G5: 7 CTAs per SM (40 registers, a few spills) hide more of phase A's load
// latency than 5 CTAs without spills: 0.270 -> 0.250 ms at K = 1, n = 32768.
// G8: likewise 5 CTAs (48 registers) over 4 (64) and 3 (80): 0.400 -> 0.376 -> 0.356 ms
// per 8 generations (the first two steps measured before the store-phase rework).
template <class M> constexpr int min_ctas() { return M::NW == 5 ? 7 : (M::NW == 6 ? 4 : 5); }

template <class M, int STRAT, bool P2P>
__global__ void __launch_bounds__(M::NT, min_ctas<M>()) ca_multi_kernel(CaArgs a) {
    __shared__ __align__(16) typename M::Smem sm;
    if (STRAT == TRI_BB) {
        if (blockIdx.x > blockIdx.y + (uint32_t)a.tile_row_begin) return;
        M::template tile<P2P>(a, blockIdx.y + (uint32_t)a.tile_row_begin, blockIdx.x, sm);
    } else if (STRAT == TRI_LAMBDA) {
        const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (w >= a.omega_end) return;
        uint32_t bi, bj;
        tri::lambda_map(w, bi, bj);
        M::template tile<P2P>(a, bi, bj, sm);
    } else {
#pragma unroll 1
        for (tri::TileWalk t(a.omega_begin, a.omega_end); t.more(); t.next()) {
            M::template tile<P2P>(a, t.bi, t.bj, sm);
            __syncthreads();                                  // smem reused by the next tile
        }
    }
}

template <class M, bool P2P>
tri_status launch_geom_p(const tri_map_t &m, int strategy, CaArgs a, cudaStream_t st) {
    constexpr int NT = M::NT;
    if (strategy == TRI_BB) {
        const int64_t tr0 = m.row_begin / m.rho;
        const int64_t tr1 = (m.row_end + m.rho - 1) / m.rho;
        if (tr1 <= tr0) return TRI_OK;
        if (tr1 - tr0 > 65535) return TRI_ENOTSUP;
        a.tile_row_begin = tr0;
        ca_multi_kernel<M, TRI_BB, P2P><<<dim3((unsigned)m.m, (unsigned)(tr1 - tr0)), NT, 0, st>>>(a);
    } else if (strategy == TRI_LAMBDA) {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        ca_multi_kernel<M, TRI_LAMBDA, P2P><<<tri::tile_grid(nb), NT, 0, st>>>(a);
    } else {
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (!nb) return TRI_OK;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ca_multi_kernel<M, TRI_LAMBDA_PERSIST, P2P>, NT, 0);
        uint64_t g = (uint64_t)tri::sm_count() * (uint64_t)(per_sm > 0 ? per_sm : 1);
        if (g > nb) g = nb;
        ca_multi_kernel<M, TRI_LAMBDA_PERSIST, P2P><<<(unsigned)g, NT, 0, st>>>(a);
    }
    tri::note_launches(1);
    return tri::cuda_status();
}

template <class M>
tri_status launch_geom(const tri_map_t &m, int strategy, CaArgs a, cudaStream_t st) {
    if (a.peer_above || a.peer_below) return launch_geom_p<M, true>(m, strategy, a, st);
    return launch_geom_p<M, false>(m, strategy, a, st);
}

// rho = 128 (k <= 16) or rho = 224 (k <= 8); the caller has validated (rho, k).
tri_status launch(const tri_map_t &m, int strategy, CaArgs a, cudaStream_t st) {
    if (m.rho == G8::RHO) return launch_geom<G8>(m, strategy, a, st);
    return a.k <= G5::KMAX ? launch_geom<G5>(m, strategy, a, st) : launch_geom<G6>(m, strategy, a, st);
}


#ifndef TRI_CA_PACKED_CTAS
#define TRI_CA_PACKED_CTAS 3
#endif
template <class M, int STRAT>
__global__ void __launch_bounds__(M::NT, TRI_CA_PACKED_CTAS) ca_packed_kernel(PackedArgs a) {
    __shared__ __align__(16) typename M::Smem sm;
    if (STRAT == TRI_BB) {
        if (blockIdx.x > blockIdx.y) return;
        M::tile_packed(a, blockIdx.y, blockIdx.x, sm);
    } else if (STRAT == TRI_LAMBDA) {
        const uint64_t w = a.omega_begin + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (w >= a.omega_end) return;
        uint32_t bi, bj;
        tri::lambda_map(w, bi, bj);
        M::tile_packed(a, bi, bj, sm);
    } else {
#pragma unroll 1
        for (tri::TileWalk t(a.omega_begin, a.omega_end); t.more(); t.next()) {
            M::tile_packed(a, t.bi, t.bj, sm);
            __syncthreads();
        }
    }
}

// bytes -> bits: word w = cells [32 w, 32 w + 32) of the packed triangle (cells >= D are 0)
__global__ void ca_pack_kernel(const uint8_t *__restrict__ in, uint64_t cells, uint32_t *__restrict__ out,
                               int64_t nwords) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nwords) return;
    const uint64_t c = 32ull * (uint64_t)w;
    uint32_t v = 0;
    if (c + 32 <= cells) {
        const uint4 *p = reinterpret_cast<const uint4 *>(in + c);
        v = bits::pack32(__ldg(p), __ldg(p + 1));
    } else {
        for (uint64_t e = 0; c + e < cells; ++e) v |= (uint32_t)(in[c + e] & 1u) << e;
    }
    out[w] = v;
}

// bits -> bytes {0, 1}
__global__ void ca_unpack_kernel(const uint32_t *__restrict__ in, uint64_t cells, uint8_t *__restrict__ out,
                                 int64_t nwords) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nwords) return;
    const uint64_t c = 32ull * (uint64_t)w;
    const uint32_t v = __ldg(in + w);
    if (c + 32 <= cells) {
        uint4 *p = reinterpret_cast<uint4 *>(out + c);
        p[0] = make_uint4(bits::spread4(v & 15u), bits::spread4((v >> 4) & 15u), bits::spread4((v >> 8) & 15u),
                          bits::spread4((v >> 12) & 15u));
        p[1] = make_uint4(bits::spread4((v >> 16) & 15u), bits::spread4((v >> 20) & 15u),
                          bits::spread4((v >> 24) & 15u), bits::spread4(v >> 28));
    } else {
        for (uint64_t e = 0; c + e < cells; ++e) out[c + e] = (uint8_t)((v >> e) & 1u);
    }
}

template <class M>
tri_status launch_packed(const tri_map_t &m, int strategy, PackedArgs a, cudaStream_t st) {
    constexpr int NT = M::NT;
    if (strategy == TRI_BB) {
        if (m.m > 65535) return TRI_ENOTSUP;
        ca_packed_kernel<M, TRI_BB><<<dim3((unsigned)m.m, (unsigned)m.m), NT, 0, st>>>(a);
    } else if (strategy == TRI_LAMBDA) {
        ca_packed_kernel<M, TRI_LAMBDA><<<tri::tile_grid(a.omega_end - a.omega_begin), NT, 0, st>>>(a);
    } else {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ca_packed_kernel<M, TRI_LAMBDA_PERSIST>, NT, 0);
        uint64_t g = (uint64_t)tri::sm_count() * (uint64_t)(per_sm > 0 ? per_sm : 1);
        const uint64_t nb = a.omega_end - a.omega_begin;
        if (g > nb) g = nb;
        ca_packed_kernel<M, TRI_LAMBDA_PERSIST><<<(unsigned)g, NT, 0, st>>>(a);
    }
    tri::note_launches(1);
    return tri::cuda_status();
}

}  // namespace multi

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
        for (tri::TileWalk t(a.omega_begin, a.omega_end); t.more(); t.next()) ca_tile<RHO>(a, t.bi, t.bj);
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
    a.k = 1;
    a.peer_above = a.peer_below = nullptr;
    a.base = m.out_offset; a.out_cells = m.out_cells;
    a.above_base = m.row_begin > 0 ? T2((uint64_t)m.row_begin - 1) : 0;
    a.omega_begin = m.omega_begin; a.omega_end = m.omega_end;
    a.tile_row_begin = 0;
    switch (m.rho) {
        case 128:                                                   // the k-generation kernel at k = 1
        case 224: return multi::launch(m, strategy, a, st);
        case 256: return bits::launch<256>(m, strategy, a, st);
        case 512: return launch_r<512>(m, strategy, a, st);
        default: return TRI_EINVAL;
    }
}

tri_status launch_ca_steps(const tri_map_t &m, int strategy, int k, const uint8_t *in, uint8_t *out,
                           const uint8_t *above, const uint8_t *below, uint8_t *peer_above, uint8_t *peer_below,
                           cudaStream_t st) {
    if (((uintptr_t)out & 15u) != 0 || ((uintptr_t)in & 15u) != 0) return TRI_EINVAL;
    CaArgs a;
    a.in = in; a.out = out;
    a.above = m.row_begin > 0 ? above : nullptr;
    a.below = m.row_end < m.n ? below : nullptr;
    a.n = m.n; a.R0 = m.row_begin; a.R1 = m.row_end;
    a.k = k;
    a.peer_above = m.row_begin > 0 ? peer_above : nullptr;
    a.peer_below = m.row_end < m.n ? peer_below : nullptr;
    a.base = m.out_offset; a.out_cells = m.out_cells;
    const int64_t first_above = m.row_begin - k > 0 ? m.row_begin - k : 0;
    a.above_base = T2((uint64_t)first_above);
    a.omega_begin = m.omega_begin; a.omega_end = m.omega_end;
    a.tile_row_begin = 0;
    return multi::launch(m, strategy, a, st);
}


size_t ca_run_ws_bytes(const tri_map_t &m) {
    const uint64_t nwords = (m.cells + 31) / 32;
    return (size_t)(2 * ((nwords * 4 + 255) / 256 * 256));
}

// steps generations at rho = 240, 8 per launch, on two packed buffers in the workspace
tri_status launch_ca_run(const tri_map_t &m, int strategy, int64_t steps, const uint8_t *in, uint8_t *out,
                         void *ws, cudaStream_t st) {
    const int64_t nwords = (int64_t)((m.cells + 31) / 32);
    const size_t half = (size_t)((nwords * 4 + 255) / 256 * 256);
    uint32_t *buf[2] = {(uint32_t *)ws, (uint32_t *)((uint8_t *)ws + half)};
    const unsigned g = (unsigned)((nwords + 255) / 256);
    multi::ca_pack_kernel<<<g, 256, 0, st>>>(in, m.cells, buf[0], nwords);
    int cur = 0;
    for (int64_t done = 0; done < steps;) {
        const int64_t k = steps - done < multi::G8P::KMAX ? steps - done : multi::G8P::KMAX;
        if (cudaMemsetAsync(buf[cur ^ 1], 0, (size_t)nwords * 4, st) != cudaSuccess) return TRI_ECUDA;
        PackedArgs a;
        a.in = buf[cur]; a.out = buf[cur ^ 1];
        a.n = m.n; a.k = k; a.nwords = nwords;
        a.omega_begin = 0; a.omega_end = m.blocks;
        const tri_status rc = multi::launch_packed<multi::G8P>(m, strategy, a, st);
        if (rc != TRI_OK) return rc;
        cur ^= 1;
        done += k;
    }
    multi::ca_unpack_kernel<<<g, 256, 0, st>>>(buf[cur], m.cells, out, nwords);
    note_launches(2);                                   // pack + unpack (launch_packed counts its own)
    return cuda_status();
}

}  // namespace tri
