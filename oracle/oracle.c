/*
 * oracle.c -- CPU ORACLE for arXiv:1609.01490 ("A Non-linear GPU Thread Map for
 * Triangular Domains", Navarro, Bustos, Hitschfeld).
 *
 * *** TEST INFRASTRUCTURE ONLY. ***
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load, call or link this file.  The product path
 * (paper_1609_01490_b200/) never touches it; the two share no code, headers,
 * tables or helpers.
 *
 * What this is: the PLAIN DEFINITION of every result the hot path computes,
 * written as double loops over the lower triangle j <= i < n (a triple loop for
 * triplets), in fp64 unless the method itself fixes the precision (the collision
 * predicate, see orc_collide).  No blocking, no tiling, no fusion, no sqrt
 * estimates: the block map lambda is obtained by enumeration (Eq. 1) or by an
 * exact integer search on the row-boundary property (Eq. 3), never by Eq. 4's
 * floating-point square root.
 *
 * Citations: "P:a-b" = /root/reference/PAPER.md lines a-b (section / equation);
 * "S:a-b" = SPEC.md lines a-b (used only for interface conventions).
 * Readings of ambiguous passages are the DESIGN.md "Readings" list (Q1..Q19).
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared oracle.c -lm
 * (-ffp-contract=off: no a*b+c contraction anywhere, so the fp32 collision
 * sequence below is exactly the one written.)
 *
 * Pins (tests/test_oracle_pins.py, -m "not gpu"): every function below is pinned
 * to something other than itself -- paper witnesses, closed forms, SPEC worked
 * examples, scipy library routines, independent algorithms, brute force.  See
 * DESIGN.md section "Oracle and its pins".
 */
#include <stdint.h>
#include <stddef.h>
#include <math.h>
#include <string.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_ERANGE (-2)

/* ------------------------------------------------------------------------ */
/* Figurate numbers.  T(r) = r(r+1)/2 (Eq. 1, the row starts of the */
/* packed layout; "sum_{r=1}^{x} r = x(x+1)/2").  T3(r) = r(r+1)(r+2)/6 */
/* (tetrahedral numbers).  Exact; overflow is an error.   */
/* ------------------------------------------------------------------------ */
int orc_tri_number(uint64_t r, uint64_t *out)
{
    unsigned __int128 v = (unsigned __int128)r * ((unsigned __int128)r + 1) / 2;
    if (v > (unsigned __int128)UINT64_MAX) return ORC_ERANGE;
    *out = (uint64_t)v;
    return ORC_OK;
}

int orc_tet_number(uint64_t r, uint64_t *out)
{
    unsigned __int128 a = (unsigned __int128)r * ((unsigned __int128)r + 1);
    /* a*(r+2) may overflow 128 bits only for r >= 2^42; reject beyond 2^40 */
    if (r > (1ull << 40)) return ORC_ERANGE;
    unsigned __int128 v = a * ((unsigned __int128)r + 2) / 6;
    if (v > (unsigned __int128)UINT64_MAX) return ORC_ERANGE;
    *out = (uint64_t)v;
    return ORC_OK;
}

static uint64_t T2(uint64_t r) { return r * (r + 1) / 2; }            /* r < 2^31 */
static uint64_t T3(uint64_t r) { return r * (r + 1) * (r + 2) / 6; }   /* r < 2^20 */

/* ------------------------------------------------------------------------ */
/* Eq. 1: blocks of the lower triangle enumerated row-major,      */
/* row i holding i+1 blocks (diag=1) -- a counter walk, no arithmetic on omega.*/
/* diag=0 enumerates the strict lower triangle (reading Q2).        */
/* Writes omega -> (I[omega], J[omega]); returns the count or <0.             */
/* ------------------------------------------------------------------------ */
int64_t orc_enumerate_tri(int64_t m, int32_t diag, uint32_t *I, uint32_t *J, uint64_t cap)
{
    if (m < 0) return ORC_EINVAL;
    uint64_t w = 0;
    for (int64_t i = 0; i < m; ++i) {
        int64_t jmax = diag ? i : i - 1;
        for (int64_t j = 0; j <= jmax; ++j) {
            if (w >= cap) return ORC_ERANGE;
            I[w] = (uint32_t)i;
            J[w] = (uint32_t)j;
            ++w;
        }
    }
    return (int64_t)w;
}

/* Tetrahedron: m stacked triangles, layer k holding the  */
/* lower triangle of side k+1, layer-major, Eq. 1 order inside each layer.     */
int64_t orc_enumerate_tet(int64_t m, uint32_t *I, uint32_t *J, uint32_t *K, uint64_t cap)
{
    if (m < 0) return ORC_EINVAL;
    uint64_t w = 0;
    for (int64_t k = 0; k < m; ++k)
        for (int64_t i = 0; i <= k; ++i)
            for (int64_t j = 0; j <= i; ++j) {
                if (w >= cap) return ORC_ERANGE;
                I[w] = (uint32_t)i; J[w] = (uint32_t)j; K[w] = (uint32_t)k;
                ++w;
            }
    return (int64_t)w;
}

/* ------------------------------------------------------------------------ */
/* lambda(omega) for ANY omega < 2^62 by the row-boundary property Eq. 3       */
/* (P:239-243): i = the largest row with T(i) <= omega, found by exact integer */
/* bisection; j = omega - T(i) (Eq. 4).  No square root.            */
/* ------------------------------------------------------------------------ */
int orc_lambda(uint64_t omega, uint32_t *bi, uint32_t *bj)
{
    if (omega >= (1ull << 62)) return ORC_ERANGE;
    uint64_t lo = 0, hi = 1ull << 32;          /* T(lo) <= omega < T(hi) */
    while (hi - lo > 1) {
        uint64_t mid = lo + (hi - lo) / 2;
        unsigned __int128 t = (unsigned __int128)mid * (mid + 1) / 2;
        if (t <= omega) lo = mid; else hi = mid;
    }
    *bi = (uint32_t)lo;
    *bj = (uint32_t)(omega - (uint64_t)((unsigned __int128)lo * (lo + 1) / 2));
    return ORC_OK;
}

/* Tetrahedral lambda (readings Q12/Q13): k = the largest layer     */
/* with T3(k) <= omega (the layer property), by exact bisection;     */
/* omega_2D = omega - T3(k); (i,j) = lambda(omega_2D).             */
int orc_tet_lambda(uint64_t omega, uint32_t *i, uint32_t *j, uint32_t *k)
{
    if (omega >= (1ull << 60)) return ORC_ERANGE;
    uint64_t lo = 0, hi = 1ull << 21;          /* T3(2^21) > 2^60 */
    while (hi - lo > 1) {
        uint64_t mid = lo + (hi - lo) / 2;
        unsigned __int128 t = (unsigned __int128)mid * (mid + 1) * (mid + 2) / 6;
        if (t <= omega) lo = mid; else hi = mid;
    }
    *k = (uint32_t)lo;
    uint64_t w2 = omega - (uint64_t)((unsigned __int128)lo * (lo + 1) * (lo + 2) / 6);
    return orc_lambda(w2, i, j);
}

/* ------------------------------------------------------------------------ */
/* Dummy kernel (reading Q6).                            */
/* PACKED: out[T(i)+j - T(row_begin)] = code(i,j) for j <= i, rows in          */
/*   [row_begin,row_end); code = (i<<16)|j as u32 when elem_bytes==4,          */
/*   (i<<32)|j as u64 when elem_bytes==8.                                      */
/* DIGEST: sum over the triangle of (i+j) ("writes the sum i+j").   */
/* ------------------------------------------------------------------------ */
int orc_dummy_packed(int64_t n, int64_t row_begin, int64_t row_end, void *out, int32_t elem_bytes)
{
    if (n < 0 || row_begin < 0 || row_end > n || row_begin > row_end) return ORC_EINVAL;
    if (elem_bytes != 4 && elem_bytes != 8) return ORC_EINVAL;
    if (elem_bytes == 4 && n > 65536) return ORC_EINVAL;
    uint64_t base = T2((uint64_t)row_begin);
    for (int64_t i = row_begin; i < row_end; ++i)
        for (int64_t j = 0; j <= i; ++j) {
            uint64_t idx = T2((uint64_t)i) + (uint64_t)j - base;
            if (elem_bytes == 4) ((uint32_t *)out)[idx] = ((uint32_t)i << 16) | (uint32_t)j;
            else ((uint64_t *)out)[idx] = ((uint64_t)i << 32) | (uint64_t)j;
        }
    return ORC_OK;
}

uint64_t orc_dummy_digest(int64_t n)
{
    uint64_t s = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j <= i; ++j) s += (uint64_t)(i + j);
    return s;
}

/* COUNT mode: emulate the dispatch of every thread the grid launches        */
/* (P:180-205 parallel spaces; P:411-418 BB discard) and count.               */
/*   strategy 0 = lambda: B = T(m) blocks, block omega -> (bi,bj) by           */
/*     ENUMERATION order (a walk over Eq. 1), thread (ty,tx) -> (bi*rho+ty,    */
/*     bj*rho+tx), useful iff j <= i < n (diag) or j < i < n (strict).         */
/*   strategy 1 = BB: m x m blocks, blocks with bx > by discarded whole,       */
/*     then the per-thread filter.                                             */
/* counts[0]=blocks dispatched, [1]=blocks discarded whole, [2]=threads        */
/* dispatched, [3]=useful threads, [4]=discarded threads.                      */
int orc_dispatch_count(int64_t n, int32_t rho, int32_t strategy, int32_t diag, uint64_t counts[5])
{
    if (n < 1 || rho < 1) return ORC_EINVAL;
    int64_t m = (n + rho - 1) / rho;
    uint64_t c[5] = {0, 0, 0, 0, 0};
    if (strategy == 0) {
        for (int64_t bi = 0; bi < m; ++bi)
            for (int64_t bj = 0; bj <= bi; ++bj) {
                c[0]++;
                for (int64_t ty = 0; ty < rho; ++ty)
                    for (int64_t tx = 0; tx < rho; ++tx) {
                        int64_t i = bi * rho + ty, j = bj * rho + tx;
                        c[2]++;
                        int ok = (i < n) && (diag ? j <= i : j < i);
                        if (ok) c[3]++; else c[4]++;
                    }
            }
    } else if (strategy == 1) {
        for (int64_t by = 0; by < m; ++by)
            for (int64_t bx = 0; bx < m; ++bx) {
                c[0]++;
                if (bx > by) { c[1]++; c[2] += (uint64_t)rho * rho; c[4] += (uint64_t)rho * rho; continue; }
                for (int64_t ty = 0; ty < rho; ++ty)
                    for (int64_t tx = 0; tx < rho; ++tx) {
                        int64_t i = by * rho + ty, j = bx * rho + tx;
                        c[2]++;
                        int ok = (i < n) && (diag ? j <= i : j < i);
                        if (ok) c[3]++; else c[4]++;
                    }
            }
    } else if (strategy == 2) {
        /* RB (reading Q19): an H x W thread rectangle, h = floor(n/2),
         * H = n - h, W = 2h + 1, tiled by rho x rho blocks; a thread is useful iff
         * it lies inside the rectangle (the fold is a bijection onto the triangle,
         * checked on the GPU by PACKED parity + COUNT). */
        int64_t h = n / 2, H = n - h, W = 2 * h + 1;
        int64_t gx = (W + rho - 1) / rho, gy = (H + rho - 1) / rho;
        for (int64_t by = 0; by < gy; ++by)
            for (int64_t bx = 0; bx < gx; ++bx) {
                c[0]++;
                for (int64_t ty = 0; ty < rho; ++ty)
                    for (int64_t tx = 0; tx < rho; ++tx) {
                        int64_t x = bx * rho + tx, y = by * rho + ty;
                        c[2]++;
                        if (x < W && y < H) c[3]++; else c[4]++;
                    }
            }
    } else return ORC_EINVAL;
    memcpy(counts, c, sizeof c);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* EDM (readings Q7/Q8).                                   */
/* out[T(i)+j - T(row_begin)] = (float) sqrt( sum_d (p_i[d] - p_j[d])^2 ),     */
/* every operation in fp64 from the fp32 inputs, rounded to fp32 once.         */
/* Points: row-major, point t at pts[t*ld .. t*ld+dim).                        */
/* ------------------------------------------------------------------------ */
int orc_edm(int64_t n, const float *pts, int32_t dim, int64_t ld,
            int64_t row_begin, int64_t row_end, float *out)
{
    if (n < 0 || dim < 1 || ld < dim || row_begin < 0 || row_end > n || row_begin > row_end)
        return ORC_EINVAL;
    uint64_t base = T2((uint64_t)row_begin);
    #pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = row_begin; i < row_end; ++i)
        for (int64_t j = 0; j <= i; ++j) {
            double s = 0.0;
            for (int32_t d = 0; d < dim; ++d) {
                double diff = (double)pts[i * ld + d] - (double)pts[j * ld + d];
                s += diff * diff;
            }
            out[T2((uint64_t)i) + (uint64_t)j - base] = (float)sqrt(s);
        }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Sphere collision count (reading Q9).                    */
/* count = #{ (i,j) : j < i, rows i in [row_begin,row_end), d2 < s*s } where,  */
/* in IEEE fp32 round-to-nearest, EXACTLY this sequence (the method's          */
/* precision, fixed by reading Q9 so both sides take the same decision):       */
/*   dx = xi - xj; dy = yi - yj; dz = zi - zj;                                 */
/*   d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));  s = ri + rj;  d2 < s * s       */
/* Spheres: 4 floats (x, y, z, r) per sphere.                                  */
/* ------------------------------------------------------------------------ */
int orc_collide(int64_t n, const float *sph, int64_t row_begin, int64_t row_end, uint64_t *count)
{
    if (n < 0 || row_begin < 0 || row_end > n || row_begin > row_end) return ORC_EINVAL;
    uint64_t total = 0;
    #pragma omp parallel for schedule(dynamic, 64) reduction(+:total)
    for (int64_t i = row_begin; i < row_end; ++i) {
        const float xi = sph[4 * i], yi = sph[4 * i + 1], zi = sph[4 * i + 2], ri = sph[4 * i + 3];
        for (int64_t j = 0; j < i; ++j) {
            float dx = xi - sph[4 * j];
            float dy = yi - sph[4 * j + 1];
            float dz = zi - sph[4 * j + 2];
            float dxx = dx * dx;
            float d2 = fmaf(dz, dz, fmaf(dy, dy, dxx));
            float s = ri + sph[4 * j + 3];
            float s2 = s * s;
            if (d2 < s2) total += 1;
        }
    }
    *count = total;
    return ORC_OK;
}

/* 1-D collision count (reading Q10): intervals          */
/* [c - r, c + r]; count = #{(i,j): j < i, |ci - cj| < ri + rj} with, in IEEE  */
/* fp32, d = ci - cj, s = ri + rj, fabsf(d) < s.  2 floats (c, r) per interval.*/
int orc_collide1d(int64_t n, const float *iv, int64_t row_begin, int64_t row_end, uint64_t *count)
{
    if (n < 0 || row_begin < 0 || row_end > n || row_begin > row_end) return ORC_EINVAL;
    uint64_t total = 0;
    #pragma omp parallel for schedule(dynamic, 64) reduction(+:total)
    for (int64_t i = row_begin; i < row_end; ++i)
        for (int64_t j = 0; j < i; ++j) {
            float d = iv[2 * i] - iv[2 * j];
            float s = iv[2 * i + 1] + iv[2 * j + 1];
            if (fabsf(d) < s) total += 1;
        }
    *count = total;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Triangular-domain cellular automaton (P:79-80 names "cellular automata     */
/* simulation on triangular domains" citing Conway's Life; reading Q11):       */
/* Life B3/S23 on the cells {(i,j): 0 <= j <= i < n}; the 8 Moore neighbours;  */
/* a neighbour outside the triangle counts as dead; synchronous update.        */
/* State: uint8 {0,1} in the packed Eq. 1 layout, in[T(i)+j].                  */
/* ------------------------------------------------------------------------ */
static int ca_alive(int64_t n, const uint8_t *s, int64_t i, int64_t j)
{
    if (i < 0 || i >= n || j < 0 || j > i) return 0;
    return s[T2((uint64_t)i) + (uint64_t)j] ? 1 : 0;
}

int orc_ca_step(int64_t n, const uint8_t *in, uint8_t *out)
{
    if (n < 0) return ORC_EINVAL;
    #pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j <= i; ++j) {
            int nb = 0;
            for (int di = -1; di <= 1; ++di)
                for (int dj = -1; dj <= 1; ++dj)
                    if (di != 0 || dj != 0) nb += ca_alive(n, in, i + di, j + dj);
            int self = ca_alive(n, in, i, j);
            out[T2((uint64_t)i) + (uint64_t)j] = (uint8_t)((nb == 3) || (self && nb == 2));
        }
    return ORC_OK;
}

/* Run `steps` generations in place (ping-pong through a scratch copy). */
int orc_ca_run(int64_t n, uint8_t *state, int64_t steps)
{
    if (n < 0 || steps < 0) return ORC_EINVAL;
    uint64_t D = T2((uint64_t)n);
    uint8_t *tmp = (uint8_t *)malloc(D ? D : 1);
    if (!tmp) return ORC_EINVAL;
    for (int64_t s = 0; s < steps; ++s) {
        orc_ca_step(n, state, tmp);
        memcpy(state, tmp, D);
    }
    free(tmp);
    return ORC_OK;
}

/* Rows [row_begin,row_end) only (bounded CPU-baseline samples); same rule.   */
int orc_ca_step_rows(int64_t n, const uint8_t *in, uint8_t *out, int64_t row_begin, int64_t row_end)
{
    if (n < 0 || row_begin < 0 || row_end > n || row_begin > row_end) return ORC_EINVAL;
    uint64_t base = T2((uint64_t)row_begin);
    #pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = row_begin; i < row_end; ++i)
        for (int64_t j = 0; j <= i; ++j) {
            int nb = 0;
            for (int di = -1; di <= 1; ++di)
                for (int dj = -1; dj <= 1; ++dj)
                    if (di != 0 || dj != 0) nb += ca_alive(n, in, i + di, j + dj);
            int self = ca_alive(n, in, i, j);
            out[T2((uint64_t)i) + (uint64_t)j - base] = (uint8_t)((nb == 3) || (self && nb == 2));
        }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Triplet-interaction energy on the tetrahedral domain (P:33-34,    */
/* P:703-704 motivate triplet n-body; the interaction itself is reading Q15:   */
/* the Axilrod-Teller-Muto three-body energy).  For a triplet with squared     */
/* side lengths a = |x_p-x_q|^2, b = |x_q-x_s|^2, c = |x_s-x_p|^2:              */
/*   E = nu * (1 + 3 cos g_p cos g_q cos g_s) / (r_pq r_qs r_sp)^3              */
/*     = nu * (1 + 3 P / (8 a b c)) / (a b c)^(3/2),                            */
/*   P = (a + c - b)(a + b - c)(b + c - a)   (law of cosines).                  */
/* Per-particle energy e_t = (1/3) * sum of E over the triplets p>q>s that     */
/* contain t.  All fp64.  Points: 4 floats per point (x, y, z, unused).        */
/* For particle t the sum runs over the unordered pairs {u,v} of the other     */
/* particles (each triplet containing t exactly once).                         */
/* Computes e[t] for t in [t_begin, t_end) only (bounded samples).             */
/* ------------------------------------------------------------------------ */
static double atm_energy(const float *P, int64_t p, int64_t q, int64_t s, double nu)
{
    double a = 0, b = 0, c = 0;
    for (int d = 0; d < 3; ++d) {
        double pq = (double)P[4 * p + d] - (double)P[4 * q + d];
        double qs = (double)P[4 * q + d] - (double)P[4 * s + d];
        double sp = (double)P[4 * s + d] - (double)P[4 * p + d];
        a += pq * pq; b += qs * qs; c += sp * sp;
    }
    double abc = a * b * c;
    double prod = (a + c - b) * (a + b - c) * (b + c - a);
    return nu * (1.0 + 3.0 * prod / (8.0 * abc)) / pow(abc, 1.5);
}

int orc_triplet(int64_t n, const float *pts, double nu, int64_t t_begin, int64_t t_end, double *e)
{
    if (n < 0 || t_begin < 0 || t_end > n || t_begin > t_end) return ORC_EINVAL;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = t_begin; t < t_end; ++t) {
        double acc = 0.0;
        for (int64_t u = 0; u < n; ++u) {
            if (u == t) continue;
            for (int64_t v = 0; v < u; ++v) {
                if (v == t) continue;
                acc += atm_energy(pts, t, u, v, nu);
            }
        }
        e[t - t_begin] = acc / 3.0;
    }
    return ORC_OK;
}

/* Per-particle absolute scale A_t = (1/3) sum |E| over the triplets containing t
 * (the normaliser of the triplet tolerance, reading Q15); same loops as above. */
int orc_triplet_abs(int64_t n, const float *pts, double nu, int64_t t_begin, int64_t t_end, double *a)
{
    if (n < 0 || t_begin < 0 || t_end > n || t_begin > t_end) return ORC_EINVAL;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = t_begin; t < t_end; ++t) {
        double acc = 0.0;
        for (int64_t u = 0; u < n; ++u) {
            if (u == t) continue;
            for (int64_t v = 0; v < u; ++v) {
                if (v == t) continue;
                acc += fabs(atm_energy(pts, t, u, v, nu));
            }
        }
        a[t - t_begin] = acc / 3.0;
    }
    return ORC_OK;
}

/* Total energy sum_{p>q>s} E (the same definition, summed once per triplet). */
int orc_triplet_total(int64_t n, const float *pts, double nu, double *total)
{
    if (n < 0) return ORC_EINVAL;
    double acc = 0.0;
    #pragma omp parallel for schedule(dynamic, 1) reduction(+:acc)
    for (int64_t p = 0; p < n; ++p)
        for (int64_t q = 0; q < p; ++q)
            for (int64_t s = 0; s < q; ++s) acc += atm_energy(pts, p, q, s, nu);
    *total = acc;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Square-root variants of Eq. 4 (section 4.1), uncorrected:       */
/*   x = 1/4 + 2 w (fp32), s = sqrt(x) by the variant, i = floor(s - 1/2)      */
/*   variant 1 (lambda_X): s = sqrtf(x) */
/*   variant 2 (lambda_N): y0 = bits(0x5f3759df - (bits(x) >> 1)), three      */
/*     Newton steps y = y (1.5 - ((x/2) y) y), s = x y + 1e-4 */
/*     -- the Carmack / Lomont code the passage cites evaluates its step as    */
/*     y * (threehalfs - (x2 * y * y)), C's left-to-right (x2 * y) * y; that   */
/*     operation order is kept (it decides the first failing omega,            */
/*     tests/golden/sqrt_variants.txt; reading Q5b).                 */
/* every operation IEEE fp32 round-to-nearest in this order (no contraction).  */
/* lambda_R (hardware rsqrt) has no bit-exact CPU definition: see            */
/* orc_variant_r_* below (its result within rsqrtf's documented error bound).  */
/* The variant is correct at w iff T(i) <= w < T(i+1) (Eq. 3).      */
/* Returns the number of failures in [w0, w0+count) and the first failing w    */
/* (UINT64_MAX if none).                                                       */
/* ------------------------------------------------------------------------ */
static uint32_t variant_row(uint64_t w, int variant)
{
    float x = 0.25f + 2.0f * (float)w;
    float s;
    if (variant == 1) {
        s = sqrtf(x);
    } else {
        float xh = 0.5f * x, y;
        int32_t bits;
        memcpy(&bits, &x, 4);
        bits = 0x5f3759df - (bits >> 1);
        memcpy(&y, &bits, 4);
        for (int it = 0; it < 3; ++it) {
            float xy2 = xh * y;
            float t = xy2 * y;
            float u = 1.5f - t;
            y = y * u;
        }
        float xy = x * y;
        s = xy + 1e-4f;
    }
    float f = floorf(s - 0.5f);
    return f > 0.0f ? (uint32_t)f : 0u;
}

int orc_variant_scan(int32_t variant, uint64_t w0, uint64_t count, uint64_t *fails, uint64_t *first)
{
    if (variant != 1 && variant != 2) return ORC_EINVAL;
    uint64_t nf = 0, fw = UINT64_MAX;
    #pragma omp parallel for schedule(static) reduction(+:nf) reduction(min:fw)
    for (uint64_t t = 0; t < count; ++t) {
        uint64_t w = w0 + t;
        uint64_t i = variant_row(w, variant);
        int ok = (T2(i) <= w) && (w < T2(i + 1));
        if (!ok) { nf += 1; if (w < fw) fw = w; }
    }
    *fails = nf;
    *first = fw;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* lambda_R: s = x * rsqrtf(x) + 1e-4, i = floor(s - 1/2), with    */
/* x = 1/4 + 2 w, every operation IEEE fp32 round-to-nearest.  rsqrtf itself    */
/* is specified only to within 2 ulp (CUDA Math API; the PTX rsqrt.approx.f32  */
/* bound 2^-22.9 is tighter), so lambda_R's row is not a single number: this    */
/* computes the rows reachable by EVERY fp32 r with |r sqrt(x) - 1| <= rel      */
/* (r bracketed outward to fp32 from the fp64 1/sqrt(x)).  The row is monotone  */
/* in r, so the reachable rows lie in [row(r_lo), row(r_hi)].  A w is SURELY    */
/* wrong when the exact row (Eq. 3) is outside that interval, MAYBE wrong when  */
/* the interval holds it and another row.  DESIGN.md reading Q5c.              */
/* ------------------------------------------------------------------------ */
static uint32_t variant_r_row(float x, float r)
{
    float xr = x * r;
    float s = xr + 1e-4f;
    float f = floorf(s - 0.5f);
    return f > 0.0f ? (uint32_t)f : 0u;
}

static void variant_r_bracket(uint64_t w, double rel, uint32_t *ilo, uint32_t *ihi)
{
    float x = 0.25f + 2.0f * (float)w;
    double q = 1.0 / sqrt((double)x);
    double qlo = q * (1.0 - rel) * (1.0 - 1e-15), qhi = q * (1.0 + rel) * (1.0 + 1e-15);
    float rlo = (float)qlo, rhi = (float)qhi;                  /* round outward to fp32 */
    if ((double)rlo > qlo) rlo = nextafterf(rlo, 0.0f);
    if ((double)rhi < qhi) rhi = nextafterf(rhi, INFINITY);
    *ilo = variant_r_row(x, rlo);
    *ihi = variant_r_row(x, rhi);
}

int orc_variant_r_rows(uint64_t w0, uint64_t count, double rel, uint32_t *ilo, uint32_t *ihi)
{
    if (!(rel >= 0.0 && rel < 1e-3)) return ORC_EINVAL;
    for (uint64_t t = 0; t < count; ++t) variant_r_bracket(w0 + t, rel, ilo + t, ihi + t);
    return ORC_OK;
}

int orc_variant_r_scan(uint64_t w0, uint64_t count, double rel, uint64_t *n_sure, uint64_t *first_sure,
                       uint64_t *n_maybe, uint64_t *first_maybe)
{
    if (!(rel >= 0.0 && rel < 1e-3)) return ORC_EINVAL;
    uint64_t ns = 0, fs = UINT64_MAX, nm = 0, fm = UINT64_MAX;
    #pragma omp parallel for schedule(static) reduction(+:ns,nm) reduction(min:fs,fm)
    for (uint64_t t = 0; t < count; ++t) {
        uint64_t w = w0 + t;
        uint32_t lo, hi;
        variant_r_bracket(w, rel, &lo, &hi);
        uint64_t i = 0;                                            /* exact row by bisection on Eq. 3 */
        uint64_t a = 0, b = 1u << 21;
        while (a < b) { uint64_t mid = (a + b + 1) / 2; if (T2(mid) <= w) a = mid; else b = mid - 1; }
        i = a;
        int sure_ok = lo == hi && lo == i;
        int sure_bad = i < lo || i > hi;
        if (!sure_ok) { nm += 1; if (w < fm) fm = w; }
        if (sure_bad) { ns += 1; if (w < fs) fs = w; }
    }
    *n_sure = ns; *first_sure = fs; *n_maybe = nm; *first_maybe = fm;
    return ORC_OK;
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count of later calls (bench.py's one-core oracle timing); k < 1: all cores. */
void orc_set_threads(int k)
{
#ifdef _OPENMP
    omp_set_num_threads(k >= 1 ? k : omp_get_num_procs());
#else
    (void)k;
#endif
}
