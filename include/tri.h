/*
 * tri.h -- C ABI of libtri.so, the B200 (sm_100a) block-space triangular map
 * lambda(omega) of Navarro, Bustos & Hitschfeld, "A Non-linear GPU Thread Map
 * for Triangular Domains" (arXiv:1609.01490), and the kernels it drives.
 *
 * Citations: "P:a-b" = PAPER.md lines a-b (section / equation / table).
 *
 * Conventions (all entry points):
 *  - Plain C types only.  Pointers named d_* are DEVICE pointers (caller-owned,
 *    e.g. torch tensors); h_* are host pointers.  The library allocates no
 *    device memory, keeps no global state except a per-device SM-count cache,
 *    and never synchronizes: every kernel call is enqueued asynchronously on
 *    `stream` (a cudaStream_t passed as void*; NULL = legacy default stream).
 *  - Argument validation is synchronous and returns a tri_status before any
 *    launch; a launch failure is reported as TRI_ECUDA (cudaGetLastError);
 *    kernel faults surface at the caller's next synchronization.
 *  - Every buffer a kernel reads or writes comes with its capacity in bytes
 *    (argument `<name>_bytes`); a capacity smaller than what the call reads or
 *    writes returns TRI_EINVAL before any launch.  The only exceptions are the
 *    peer-memory destinations of tri_ca_steps_p2p (addresses in another
 *    process's allocation, sized by the owner) and the map self-check hooks.
 *  - Indices: cells (i, j) of the lower triangle 0 <= j <= i < n (P:86-87,
 *    P:189-199).  The PACKED layout of Eq. 1 stores cell (i, j) at T(i) + j,
 *    T(i) = i(i+1)/2; a rank's slice stores it at T(i) + j - out_offset.
 *  - Strategies (every kernel has all three, P:411-418 for BB):
 *      TRI_LAMBDA          one CTA per tile omega, 1-D grid of B tiles, tile
 *                          coordinate = lambda(omega) (Eq. 4);
 *      TRI_BB              m x m grid, tiles above the diagonal exit on a
 *                          block test, diagonal tiles filter per thread;
 *      TRI_LAMBDA_PERSIST  a grid of (SMs x resident CTAs) CTAs, each walking
 *                          a contiguous omega chunk: lambda once at the chunk
 *                          start, then the Eq. 1 successor rule;
 *      TRI_LAMBDA_CLC      (tri_edm only) the TRI_LAMBDA grid run by
 *                          persistent CTAs that take further tiles by
 *                          cancelling not-yet-launched CTAs (sm_100 cluster
 *                          launch control), lambda per tile.
 */
#ifndef TRI_H_
#define TRI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TRI_OK = 0,
    TRI_EINVAL = -1,  /* bad argument, NULL pointer, unsupported rho, buffer too small */
    TRI_ERANGE = -2,  /* 64-bit capacity or the 2^40 omega bound exceeded              */
    TRI_ECUDA = -3,   /* CUDA launch / runtime error                                   */
    TRI_ENOTSUP = -4  /* valid request this build does not implement                   */
} tri_status;

enum { TRI_LAMBDA = 0, TRI_BB = 1, TRI_LAMBDA_PERSIST = 2, TRI_LAMBDA_CLC = 7 };
/* tri_collide only, rho = 128 k for k = 2..8 (256 and 512 are also SIMT tile edges; the others
 * belong to these strategies only): the filter gap
 * evaluated on the 5th-generation tensor cores (one tcgen05.mma.kind::f16 per 128 x 128
 * block into an F16 TMEM accumulator, csrc/collide_tc.cu); the count is the same exact
 * fixed-order predicate (reading Q9).
 * TRI_LAMBDA_TC runs the TRI_LAMBDA grid (one CTA per tile omega), TRI_BB_TC the same
 * tile body on the m x m BB grid -- the like-for-like comparator. */
enum { TRI_LAMBDA_TC = 8, TRI_BB_TC = 9 };
/* The paper's square-root variants of Eq. 4 (section 4.1), used WITHOUT
 * the integer correction: lambda_X = IEEE sqrtf, lambda_N = 0x5f3759df seed + 3
 * Newton steps + eps, lambda_R = x * rsqrtf(x) + eps, eps = 1e-4.  Exact only
 * inside their validity range (see tri_map_eval_variant).  Accepted as a
 * strategy by tri_dummy only (the map-cost experiment of Fig. 2). */
enum { TRI_LAMBDA_X = 3, TRI_LAMBDA_N = 4, TRI_LAMBDA_R = 5 };
/* RB, the rectangular-box comparator (reading Q19): the triangle folded
 * into an H x W thread rectangle, h = n/2, H = n - h, W = 2h + 1, one thread per
 * cell.  Accepted by tri_dummy and tri_edm, single rank (world = 1) only. */
enum { TRI_RB = 6 };
enum { TRI_SQRT_X = 1, TRI_SQRT_N = 2, TRI_SQRT_R = 3 };
enum { TRI_DUMMY_FIXED = 0, TRI_DUMMY_PACKED = 1, TRI_DUMMY_DIGEST = 2, TRI_DUMMY_COUNT = 3 };

/* Exactness bound of the device lambda: omega < 2^40 (checked exhaustively). */
#define TRI_OMEGA_MAX (1ull << 40)

/*
 * Triangular-domain map descriptor.  Filled by tri_map_init; read-only
 * afterwards; may be copied freely.
 *   n            linear size of the domain (rows), n >= 1
 *   rho          tile edge in cells ("dimensional block size")
 *   diag         1: cells j <= i (D = n(n+1)/2); 0: strict j < i (D = n(n-1)/2)
 *   rank, world  this process's share of a world-way partition (one GPU each)
 *   m            ceil(n / rho) tiles per dimension
 *   blocks       B = T(m) = m(m+1)/2 lambda tiles (Eq. 1)
 *   cells        D (whole domain)
 *   omega_begin, omega_end   this rank's lambda tile range [begin, end)
 *   row_begin, row_end       this rank's cell rows [begin, end) (snapped to tile rows)
 *   out_offset, out_cells    packed slice [T(row_begin), T(row_end)) of Eq. 1
 *   waste_lambda, waste_bb   closed-form unnecessary threads of a whole-domain
 *                            launch with one thread per cell: B rho^2 - D and
 *                            m^2 rho^2 - D
 *   snap         1: omega range = [T(R_g), T(R_g+1)), R_g the tile row minimising
 *                |T(R) - g B / world| (lambda applied at partition level);
 *                0: omega range = [floor(g B / world), floor((g+1) B / world))
 */
typedef struct {
    int64_t n;
    int32_t rho, diag, rank, world;
    int64_t m;
    uint64_t blocks, cells;
    uint64_t omega_begin, omega_end;
    int64_t row_begin, row_end;
    uint64_t out_offset, out_cells;
    uint64_t waste_lambda, waste_bb;
    int32_t snap, reserved;
} tri_map_t;

/* P:180-205.  EINVAL: n < 1, rho < 1 or > 1024, world < 1, rank outside
 * [0, world); ERANGE: T(m) >= 2^40 or T(n) overflows. */
tri_status tri_map_init(tri_map_t *map, int64_t n, int32_t rho, int32_t diag,
                        int32_t rank, int32_t world, int32_t snap_rows);

/* Host mirror of the device map, Eq. 4 with the integer
 * correction of the row-boundary property Eq. 3:
 * (bi, bj) = (largest i with T(i) <= omega, omega - T(i)).  ERANGE: omega >= 2^40. */
tri_status tri_lambda(uint64_t omega, uint32_t *bi, uint32_t *bj);

/* Eq. 5, the map onto the strict lower triangle, with its garbled
 * j-term corrected (reading Q2): (i, j) = (lambda(omega).i + 1, lambda(omega).j),
 * i.e. i = floor(sqrt(1/4 + 2 omega) + 1/2), j = omega - i(i-1)/2.  Host mirror
 * of the device function tri_collide1d uses.  ERANGE: omega >= 2^40. */
tri_status tri_lambda_nodiag(uint64_t omega, uint32_t *i, uint32_t *j);

/* GPU self-check of the map on omega in [omega0, omega0 + count):
 * counts on device (into *d_fail, u64, zeroed by the call) every omega whose
 * lambda violates Eq. 3 (T(i) <= omega < T(i+1)) or the Eq. 1 successor rule
 * lambda(omega+1) in {(i, j+1), (i+1, 0)}.  If d_ij != NULL also writes
 * d_ij[2t] = i, d_ij[2t+1] = j for t < count (requires count < 2^31).
 * ERANGE: omega0 + count > 2^40. */
tri_status tri_map_eval(uint64_t omega0, uint64_t count, uint32_t *d_ij,
                        unsigned long long *d_fail, void *stream);

/* Validity scan of a square-root variant (TRI_SQRT_X / _N / _R) on omega in
 * [omega0, omega0 + count): *d_fail (u64, zeroed by the call) = number of omega
 * whose uncorrected variant differs from the exact lambda; *d_first (u64, set to
 * UINT64_MAX by the call) = smallest such omega.  Reproduces the paper's
 * "valid in N in [0, 30720]" claim on this hardware.
 * EINVAL: bad variant; ERANGE: omega0 + count > 2^40. */
tri_status tri_map_eval_variant(int32_t variant, uint64_t omega0, uint64_t count,
                                unsigned long long *d_fail, unsigned long long *d_first, void *stream);

/* Rows of a square-root variant (TRI_SQRT_X / _N / _R), uncorrected: d_rows[t] (u32,
 * rows_bytes >= 4 count, 4-byte aligned) = the variant's row i at omega0 + t, i.e.
 * floor(sqrt_variant(1/4 + 2 omega) - 1/2) in fp32.  lambda_R's row depends
 * on the hardware rsqrtf, which is specified only to 2 ulp: tests check these rows
 * against the oracle's reachable-row interval (reading Q5c).
 * EINVAL: bad variant / pointer / capacity; ERANGE: omega0 + count > 2^40. */
tri_status tri_map_rows_variant(int32_t variant, uint64_t omega0, uint64_t count, uint32_t *d_rows,
                                size_t rows_bytes, void *stream);

/* Dummy kernel: each useful thread maps itself to (i,j).
 *   FIXED  : writes i + j to d_out[0] (u32; racy by design)
 *   PACKED : d_out[T(i)+j - out_offset] = (i<<16)|j as u32 when n <= 65536, else
 *            (i<<32)|j as u64; needs out_cells * elem bytes.  Requires diag = 1.
 *   DIGEST : *(u64*)d_out = sum over this rank's cells of (i + j) (zeroed by call)
 *   COUNT  : 5 x u64 (zeroed by call): tiles dispatched, tiles discarded whole,
 *            threads dispatched, useful threads, discarded threads.
 * One thread per cell, rho x rho threads per CTA: rho in {8, 16, 32}. */
tri_status tri_dummy(const tri_map_t *map, int32_t strategy, int32_t mode,
                     void *d_out, size_t out_bytes, void *stream);

/* Euclidean distance matrix: for this rank's packed slice,
 * d_out[T(i)+j - out_offset] = || p_i - p_j ||_2 in fp32 for j <= i (diag = 1).
 * d_pts: n points, point t at d_pts[t*ld .. t*ld+dim), dim in 1..4, ld >= dim;
 * pts_bytes >= 4 * ((n-1)*ld + dim).  Requires out_bytes >= 4 * out_cells, d_out
 * 16-byte aligned (32 at rho = 256); rho in {32,64,128,256}; strategy TRI_LAMBDA,
 * TRI_BB, TRI_LAMBDA_PERSIST, TRI_LAMBDA_CLC or TRI_RB (world = 1); world > 1
 * needs a snapped map (the rank's slice is contiguous).  Stores are aligned
 * 16-byte streaming stores; each 16-byte chunk of the slice is written by exactly
 * one thread (at rho = 128 each 128-byte line of the slice by one warp store, so a
 * 128-byte-aligned d_out gives whole-line writes). */
tri_status tri_edm(const tri_map_t *map, int32_t strategy, const float *d_pts,
                   int32_t dim, int64_t ld, size_t pts_bytes, float *d_out, size_t out_bytes,
                   void *stream);

/* Host-buffer EDM (end-to-end through the ABI): the same result as tri_edm with
 * h_pts / h_out HOST buffers (pinned for overlap).  The points are uploaded to
 * the caller's device buffer d_pts_ws (pts_ws_bytes >= 4 * n * ld); the packed
 * output is produced in row bands (whole tile rows) of at most band_cells cells
 * (0: as large as the workspace allows) into two halves of the caller's device
 * workspace d_ws (32-byte aligned), and each band is copied to h_out while the
 * next one is computed (two CUDA streams created and destroyed by the call).
 * Synchronous: returns when h_out is complete.  Validation is tri_edm's
 * (map, strategy -- TRI_RB excepted --, rho, dim, ld, pts_bytes = the host
 * buffer's capacity, out_bytes = h_out's), plus: EINVAL when one tile row of
 * the slice (rho rows, <= rho * row_end cells) does not fit one half of d_ws or
 * in band_cells. */
tri_status tri_edm_host(const tri_map_t *map, int32_t strategy, const float *h_pts,
                        int32_t dim, int64_t ld, size_t pts_bytes, float *d_pts_ws,
                        size_t pts_ws_bytes, float *h_out, size_t out_bytes, void *d_ws,
                        size_t ws_bytes, uint64_t band_cells);

/* Sphere collision count: *d_count (u64, zeroed by call) =
 * number of pairs j < i in this rank's omega tiles with
 *   d2 = fma(dz,dz, fma(dy,dy, dx*dx)) < (ri + rj)^2
 * evaluated in IEEE fp32 round-to-nearest with exactly that operation order.
 * d_spheres: n x 4 floats (x, y, z, r), 16-byte aligned, spheres_bytes >= 16 n.
 * count_bytes >= 8.  rho in {128,256,512} (SIMT strategies) or 128 k, k = 2..8 (tensor-core
 * strategies).
 * The map must be built with diag = 1 (tiles) -- the strict filter is per pair.
 * TRI_LAMBDA_TC / TRI_BB_TC need d_ws (tri_collide_workspace_size bytes, 16-byte
 * aligned).  If a tensor-core or bulk-copy completion ever fails to arrive within ~2 s
 * (it never should) the kernel sets bit 63 of *d_count and traps: the launch fails
 * (TRI_ECUDA / a CUDA error at the next synchronization) and the count is marked
 * invalid -- a real pair count is < 2^63. */
tri_status tri_collide(const tri_map_t *map, int32_t strategy, const float *d_spheres,
                       size_t spheres_bytes, unsigned long long *d_count, size_t count_bytes,
                       void *d_ws, size_t ws_bytes, void *stream);

/* Device workspace tri_collide needs for `strategy` (bytes, 16-byte aligned; 0 for the
 * SIMT strategies, which accept d_ws = NULL).  TRI_LAMBDA_TC / TRI_BB_TC: 256 + m * rho * 64
 * bytes -- a header (the coordinate bound that picks the power-of-two scale) and the
 * fp16 row and column operands of every sphere (plus pad rows), written by the call's
 * first kernels and read by the tiles with bulk (TMA) copies. */
size_t tri_collide_workspace_size(const tri_map_t *map, int32_t strategy);

/* Test hook: D = X Y^T (128 x 128, fp32, row-major) from ONE tcgen05.mma.kind::tf32
 * 128 x 128 x 8 with the caller's operands (row-major 128 x 8 fp32, used as TF32: the
 * low 13 mantissa bits are ignored).  It exposes the tensor core's fp32 accumulation
 * error, which the TRI_LAMBDA_TC filter's margin assumes bounded by 2^-20 sum |x y|. */
tri_status tri_tc_tf32_probe(const float *d_x, const float *d_y, float *d_d, void *stream);

/* Test hook: D (128 x 128 fp16 bit patterns, row-major) = X Y^T from ONE
 * tcgen05.mma.kind::f16 128 x 128 x 16 with the caller's fp16 operands (row-major
 * 128 x 16) into an F16 accumulator, read back with the packed 16-bit TMEM loads the
 * collision filter uses.  The filter assumes the accumulator holds the correctly rounded
 * value of a wide (>= fp32) sum of the products. */
tri_status tri_tc_f16_probe(const void *d_x, const void *d_y, void *d_d, void *stream);

/* 1-D collision count (reading Q10): *d_count (u64, zeroed by
 * the call) = number of pairs j < i with |c_i - c_j| < r_i + r_j, evaluated in IEEE
 * fp32 as d = ci - cj, s = ri + rj, |d| < s.  d_intervals: n x 2 floats (c, r),
 * 8-byte aligned, intervals_bytes >= 8 n; count_bytes >= 8.  rho = 256.  TRI_LAMBDA
 * launches the T(m-1) strictly-lower tiles through Eq. 5 (tri_lambda_nodiag) then
 * the m diagonal tiles; TRI_BB the m x m grid.  Ranks split the T(m) tiles by the
 * plain omega range (lambda) or by the map's snapped tile rows (BB). */
tri_status tri_collide1d(const tri_map_t *map, int32_t strategy, const float *d_intervals,
                         size_t intervals_bytes, unsigned long long *d_count, size_t count_bytes,
                         void *stream);

/* Device workspace tri_ca_step needs (bytes; may be 0). */
size_t tri_ca_workspace_size(const tri_map_t *map);

/* One synchronous generation of Life B3/S23 on the triangle (the
 * rule is Conway's, cells outside the triangle dead).  d_in/d_out: this rank's
 * packed slice (in_bytes, out_bytes >= out_cells; u8 {0,1}, 16-byte aligned,
 * must not alias).  d_halo_above = row row_begin-1 (above_bytes >= row_begin)
 * or NULL (dead); d_halo_below = row row_end (below_bytes >= row_end + 1) or
 * NULL (dead; ignored when row_end == n).  rho (tile edge) in {128, 224, 256,
 * 512}.  d_ws: tri_ca_workspace_size bytes (NULL if 0). */
tri_status tri_ca_step(const tri_map_t *map, int32_t strategy, const uint8_t *d_in,
                       size_t in_bytes, uint8_t *d_out, size_t out_bytes,
                       const uint8_t *d_halo_above, size_t above_bytes,
                       const uint8_t *d_halo_below, size_t below_bytes, void *d_ws, void *stream);

/* k generations of the same rule in one call (temporal blocking, deep halos;
 * k in 1..16 at rho = 128, 1..8 at rho = 224): d_out = the state after k generations of the whole
 * domain restricted to this rank's slice, given the current state of the
 * rank's rows (d_in) and of the k rows on either side.  d_halo_above = the
 * packed rows [max(row_begin - k, 0), row_begin) (contiguous in the owner's
 * slice) or NULL when row_begin == 0; d_halo_below = the packed rows
 * [row_end, min(row_end + k, n)) or NULL when row_end == n.  Capacities:
 * in_bytes, out_bytes >= out_cells; above_bytes >= T(row_begin) -
 * T(max(row_begin - k, 0)); below_bytes >= T(min(row_end + k, n)) - T(row_end)
 * (unchecked for a NULL halo).  Each tile writes only its own cells (partial
 * 16-byte chunks byte-wise).  k = 1 computes the same result as tri_ca_step.
 * HBM traffic per cell-generation ~2.2/k bytes. */
tri_status tri_ca_steps(const tri_map_t *map, int32_t strategy, int32_t k, const uint8_t *d_in,
                        size_t in_bytes, uint8_t *d_out, size_t out_bytes,
                        const uint8_t *d_halo_above, size_t above_bytes,
                        const uint8_t *d_halo_below, size_t below_bytes, void *d_ws, void *stream);

/* tri_ca_steps with the halo exchange fused into the kernel's store phase
 * (peer-memory halo stores over NVLink instead of a
 * separate send/recv after the kernel).  Same arguments and result as
 * tri_ca_steps, plus two destinations the tiles ALSO store to while writing
 * d_out:
 *   d_peer_above: the packed rows [row_begin, row_begin + k) of the NEW state,
 *     at offsets [0, T(row_begin + k) - T(row_begin)) -- i.e. the halo_below
 *     buffer of the rank owning row row_begin - 1 (ignored when row_begin == 0);
 *   d_peer_below: a base address such that the packed rows [row_end - k, row_end)
 *     land at d_peer_below + (T(r) + c - T(row_begin)) -- i.e. the halo_above
 *     buffer of the rank owning row row_end sits at d_peer_below +
 *     T(row_end - k) - T(row_begin) (ignored when row_end == n).
 * Both 16-byte aligned (EINVAL otherwise), device pointers valid in this
 * context (peer memory opened with tri_ipc_open, or local buffers), or NULL.
 * A rank owning rows must own >= k of them (EINVAL).  The stores are ordinary
 * global stores: the caller orders them against the peers' next launch (e.g. a
 * stream-ordered 4-byte all-reduce per epoch) and double-buffers the halo
 * buffers by epoch parity so a launch never writes a buffer a peer still reads. */
tri_status tri_ca_steps_p2p(const tri_map_t *map, int32_t strategy, int32_t k, const uint8_t *d_in,
                            size_t in_bytes, uint8_t *d_out, size_t out_bytes,
                            const uint8_t *d_halo_above, size_t above_bytes,
                            const uint8_t *d_halo_below, size_t below_bytes,
                            uint8_t *d_peer_above, uint8_t *d_peer_below, void *d_ws, void *stream);

/* `steps` generations of the same rule over the whole domain (world = 1, diag = 1,
 * rho = 240), bytes in, bytes out: the state is packed to bits once (cell (i, j) at bit
 * T(i) + j), advanced 8 generations per launch on two packed buffers in d_ws
 * (tri_ca_run_workspace_size bytes: 2 x ceil(D / 32) words, 256-byte rounded; 16-byte
 * aligned) -- a tile loads its region's covering words, keeps the generations in
 * registers, stores whole words and OR-merges the partial words it shares with a
 * neighbouring tile or row (the launch's output buffer is zeroed first) -- and unpacked
 * once.  d_in / d_out: the packed Eq. 1 uint8 {0,1} state, in_bytes, out_bytes >= D,
 * 16-byte aligned, may alias.  Same result as steps / 8 calls of tri_ca_steps; 8x less
 * HBM traffic per launch than the byte state. */
size_t tri_ca_run_workspace_size(const tri_map_t *map);
tri_status tri_ca_run(const tri_map_t *map, int32_t strategy, int64_t steps, const uint8_t *d_in,
                      size_t in_bytes, uint8_t *d_out, size_t out_bytes, void *d_ws, size_t ws_bytes,
                      void *stream);

/* CUDA IPC for the peer buffers of tri_ca_steps_p2p (one process per GPU).
 * tri_ipc_handle: the TRI_IPC_HANDLE_BYTES-byte handle of the device allocation
 * holding d_ptr and d_ptr's offset in it (cudaIpcGetMemHandle on the allocation
 * base).  tri_ipc_open: maps a handle from another process (peer access enabled
 * lazily); *d_ptr = base + offset, *d_base = the mapping to pass to tri_ipc_close.
 * ECUDA on any CUDA failure (e.g. a handle opened in the process that made it). */
#define TRI_IPC_HANDLE_BYTES 64
tri_status tri_ipc_handle(const void *d_ptr, void *handle, uint64_t *offset);
tri_status tri_ipc_open(const void *handle, uint64_t offset, void **d_ptr, void **d_base);
tri_status tri_ipc_close(void *d_base);

/*
 * Tetrahedral map descriptor.  Tiles (i, j, k), j <= i <= k < m,
 * enumerated layer-major (layer k = a triangle of side k+1, Eq. 1 inside).
 *   blocks = T3(m) = m(m+1)(m+2)/6; rank's tile range [omega_begin, omega_end).
 */
typedef struct {
    int64_t n;
    int32_t rho, rank, world, reserved;
    int64_t m;
    uint64_t blocks, omega_begin, omega_end;
    uint64_t waste_tet, waste_bb;  /* unnecessary threads (one per cell, strict p>q>s) */
} tet_map_t;

/* EINVAL: n < 3, rho not in {4, 8, 16, 32} (kernels: 8, 16, 32), bad rank/world. ERANGE: T3(m) >= 2^40. */
tri_status tet_map_init(tet_map_t *map, int64_t n, int32_t rho, int32_t rank, int32_t world);

/* Host mirror of the tetrahedral map (P:617-654 with integer correction):
 * k = largest layer with T3(k) <= omega, (i, j) = lambda(omega - T3(k)). */
tri_status tet_lambda(uint64_t omega, uint32_t *i, uint32_t *j, uint32_t *k);

/* GPU self-check of the tetrahedral map on [omega0, omega0+count): failures of
 * T3(k) <= omega < T3(k+1), j <= i <= k, and the layer-major successor rule. */
tri_status tet_map_eval(uint64_t omega0, uint64_t count, uint32_t *d_ijk,
                        unsigned long long *d_fail, void *stream);

/* Succinct lookup table for the tetrahedral layer index ("a succint
 * lookup table of o(T_n) combined with coordinate computations"; it deliberately
 * relaxes the paper's no-extra-data condition, P:405-410 -- SURVEY 8(f)4).
 * Layers k = 0..kmax.  Layout of the caller-owned device buffer (8-byte aligned):
 *   S[k] = T3(k), k = 0..kmax+1                                  (uint64)
 *   G[g] = max{k : T3(k) <= g * 2^shift}, g = 0..nb, nb = (T3(kmax+1) >> shift) + 1  (uint32)
 * k(omega) = the largest k in [G[g], G[g+1]] with S[k] <= omega, g = omega >> shift
 * (a bisection over the few layers of one bucket), then (i, j) = lambda(omega - S[k]):
 * loads instead of the cube root.  shift in [0, 40]; 0 < kmax < 2^20.
 * tet_lut_bytes: buffer size (0 on bad arguments).  tet_lut_build: fills the buffer on
 * the stream.  tet_map_eval_lut: tet_map_eval with the table-based map; requires
 * omega0 + count < T3(kmax+1) (TRI_ERANGE otherwise). */
size_t tet_lut_bytes(uint32_t kmax, int32_t shift);
tri_status tet_lut_build(uint32_t kmax, int32_t shift, void *d_lut, size_t lut_bytes, void *stream);
tri_status tet_map_eval_lut(uint64_t omega0, uint64_t count, uint32_t kmax, int32_t shift, const void *d_lut,
                            uint32_t *d_ijk, unsigned long long *d_fail, void *stream);

/* Triplet-interaction n-body on the tetrahedral map (
 * interaction = Axilrod-Teller-Muto, reading Q15): for every
 * triplet p > q > s in this rank's tiles, E = nu (1 + 3P/(8abc)) / (abc)^(3/2)
 * with a = |x_p-x_q|^2, b = |x_q-x_s|^2, c = |x_s-x_p|^2,
 * P = (a+c-b)(a+b-c)(b+c-a); d_energy[t] (n doubles, zeroed by the call) +=
 * E/3 for t in {p, q, s}.  Terms in fp32, accumulation in fp64.
 * d_pts4: n x 4 floats (x, y, z, unused), 16-byte aligned, pts_bytes >= 16 n;
 * energy_bytes >= 8 n. */
tri_status tet_triplet(const tet_map_t *map, int32_t strategy, const float *d_pts4,
                       size_t pts_bytes, double nu, double *d_energy, size_t energy_bytes,
                       void *stream);

/* Number of kernels the most recent successful call on this host thread
 * enqueued (for the bench's launch accounting). */
int32_t tri_last_launch_count(void);

const char *tri_status_str(tri_status s);

#ifdef __cplusplus
}
#endif
#endif /* TRI_H_ */
