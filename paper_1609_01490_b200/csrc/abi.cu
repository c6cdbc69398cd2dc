// abi.cu -- the C ABI of libtri.so (include/tri.h): descriptors, partition
// arithmetic, validation and dispatch to the kernel launchers.
#include <cstring>
#include "tri_common.cuh"

namespace tri {

static thread_local int g_launches = 0;
void note_launches(int k) { g_launches += k; }
void reset_launches() { g_launches = 0; }

int sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            v = 148;
        cache[dev] = v;
    }
    return cache[dev];
}

// |world * T(r) - g * B| as unsigned 128-bit (partition snapping, reading Q17)
static unsigned __int128 snap_dist(uint64_t r, uint64_t g, uint64_t B, uint64_t world) {
    unsigned __int128 a = (unsigned __int128)world * T2(r);
    unsigned __int128 b = (unsigned __int128)g * B;
    return a > b ? a - b : b - a;
}

// Tile row R_g minimising |T(R) - g B / world|; ties -> the smaller row.
static uint64_t snap_row(uint64_t g, uint64_t world, uint64_t m, uint64_t B) {
    if (g == 0) return 0;
    if (g >= world) return m;
    uint64_t target = (uint64_t)(((unsigned __int128)g * B) / world);
    uint32_t r, c;
    lambda_map(target, r, c);        // lambda applied at partition level
    uint64_t best = r;
    if (r + 1 <= m && snap_dist(r + 1, g, B, world) < snap_dist(r, g, B, world)) best = r + 1;
    return best > m ? m : best;
}

// [base, base + size) of the device allocation holding p (cuMemGetAddressRange,
// resolved through the runtime so the library needs no link-time libcuda).
static tri_status cuda_driver_range(const void *p, void **base, size_t *size) {
    typedef int (*range_fn)(unsigned long long *, size_t *, unsigned long long);
    static range_fn fn = nullptr;
    if (!fn) {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !f)
            return TRI_ECUDA;
        fn = (range_fn)f;
    }
    unsigned long long b = 0;
    if (fn(&b, size, (unsigned long long)(uintptr_t)p) != 0) return TRI_ECUDA;
    *base = (void *)(uintptr_t)b;
    return TRI_OK;
}

}  // namespace tri

using namespace tri;

extern "C" {

tri_status tri_map_init(tri_map_t *map, int64_t n, int32_t rho, int32_t diag, int32_t rank,
                        int32_t world, int32_t snap_rows) {
    if (!map || n < 1 || rho < 1 || rho > 1024 || world < 1 || rank < 0 || rank >= world)
        return TRI_EINVAL;
    if (n > (int64_t)(1ll << 31)) return TRI_ERANGE;
    tri_map_t t;
    std::memset(&t, 0, sizeof t);
    t.n = n; t.rho = rho; t.diag = diag ? 1 : 0; t.rank = rank; t.world = world;
    t.snap = snap_rows ? 1 : 0;
    t.m = (n + rho - 1) / rho;
    const uint64_t m = (uint64_t)t.m;
    t.blocks = T2(m);
    if (t.blocks >= TRI_OMEGA_MAX) return TRI_ERANGE;
    t.cells = t.diag ? T2((uint64_t)n) : T2((uint64_t)n - 1);
    const uint64_t R0 = snap_row((uint64_t)rank, (uint64_t)world, m, t.blocks);
    const uint64_t R1 = snap_row((uint64_t)rank + 1, (uint64_t)world, m, t.blocks);
    t.row_begin = (int64_t)(R0 * (uint64_t)rho);
    t.row_end = (int64_t)(R1 * (uint64_t)rho);
    if (t.row_begin > n) t.row_begin = n;
    if (t.row_end > n) t.row_end = n;
    if (t.snap) {
        t.omega_begin = T2(R0);
        t.omega_end = T2(R1);
    } else {
        t.omega_begin = (uint64_t)(((unsigned __int128)rank * t.blocks) / (uint64_t)world);
        t.omega_end = (uint64_t)(((unsigned __int128)(rank + 1) * t.blocks) / (uint64_t)world);
    }
    t.out_offset = T2((uint64_t)t.row_begin);
    t.out_cells = T2((uint64_t)t.row_end) - t.out_offset;
    const uint64_t r2 = (uint64_t)rho * (uint64_t)rho;
    t.waste_lambda = t.blocks * r2 - t.cells;
    t.waste_bb = m * m * r2 - t.cells;
    *map = t;
    return TRI_OK;
}

tri_status tri_lambda(uint64_t omega, uint32_t *bi, uint32_t *bj) {
    if (!bi || !bj) return TRI_EINVAL;
    if (omega >= TRI_OMEGA_MAX) return TRI_ERANGE;
    lambda_map(omega, *bi, *bj);
    return TRI_OK;
}

tri_status tri_map_eval(uint64_t omega0, uint64_t count, uint32_t *d_ij, unsigned long long *d_fail,
                        void *stream) {
    g_launches = 0;
    if (!d_fail) return TRI_EINVAL;
    if (omega0 > TRI_OMEGA_MAX || count > TRI_OMEGA_MAX - omega0) return TRI_ERANGE;
    if (d_ij && count >= (1ull << 31)) return TRI_EINVAL;
    return launch_map_eval(omega0, count, d_ij, d_fail, (cudaStream_t)stream);
}

static bool bad_map(const tri_map_t *m);

tri_status tri_lambda_nodiag(uint64_t omega, uint32_t *i, uint32_t *j) {
    if (!i || !j) return TRI_EINVAL;
    if (omega >= TRI_OMEGA_MAX) return TRI_ERANGE;
    lambda_nodiag(omega, *i, *j);
    return TRI_OK;
}

tri_status tri_collide1d(const tri_map_t *map, int32_t strategy, const float *d_intervals,
                         size_t intervals_bytes, unsigned long long *d_count, size_t count_bytes,
                         void *stream) {
    g_launches = 0;
    if (bad_map(map) || (strategy != TRI_LAMBDA && strategy != TRI_BB) || !d_intervals || !d_count)
        return TRI_EINVAL;
    if (map->rho != 256 || (((uintptr_t)d_intervals) & 7u)) return TRI_EINVAL;
    if (intervals_bytes / 8u < (uint64_t)map->n || count_bytes < 8 || (((uintptr_t)d_count) & 7u))
        return TRI_EINVAL;
    return launch_collide1d(*map, strategy, d_intervals, d_count, (cudaStream_t)stream);
}

tri_status tri_map_eval_variant(int32_t variant, uint64_t omega0, uint64_t count, unsigned long long *d_fail,
                                unsigned long long *d_first, void *stream) {
    g_launches = 0;
    if (!d_fail || !d_first || variant < TRI_SQRT_X || variant > TRI_SQRT_R) return TRI_EINVAL;
    if (omega0 > TRI_OMEGA_MAX || count > TRI_OMEGA_MAX - omega0) return TRI_ERANGE;
    return launch_variant_scan(variant, omega0, count, d_fail, d_first, (cudaStream_t)stream);
}

tri_status tri_map_rows_variant(int32_t variant, uint64_t omega0, uint64_t count, uint32_t *d_rows,
                                size_t rows_bytes, void *stream) {
    g_launches = 0;
    if (!d_rows || (((uintptr_t)d_rows) & 3u) || variant < TRI_SQRT_X || variant > TRI_SQRT_R) return TRI_EINVAL;
    if (omega0 > TRI_OMEGA_MAX || count > TRI_OMEGA_MAX - omega0) return TRI_ERANGE;
    if (rows_bytes / 4u < count) return TRI_EINVAL;
    return launch_variant_rows(variant, omega0, count, d_rows, (cudaStream_t)stream);
}

static bool bad_strategy(int32_t s) { return s != TRI_LAMBDA && s != TRI_BB && s != TRI_LAMBDA_PERSIST; }

static bool bad_map(const tri_map_t *m) {
    return !m || m->n < 1 || m->rho < 1 || m->m != (m->n + m->rho - 1) / m->rho ||
           m->blocks != T2((uint64_t)m->m) || m->omega_end < m->omega_begin ||
           m->omega_end > m->blocks || m->row_begin < 0 || m->row_end > m->n ||
           m->row_begin > m->row_end;
}

tri_status tri_dummy(const tri_map_t *map, int32_t strategy, int32_t mode, void *d_out,
                     size_t out_bytes, void *stream) {
    g_launches = 0;
    const bool extra = (strategy >= TRI_LAMBDA_X && strategy <= TRI_LAMBDA_R) || strategy == TRI_RB;
    if (bad_map(map) || (bad_strategy(strategy) && !extra) || !d_out) return TRI_EINVAL;
    if (map->rho != 8 && map->rho != 16 && map->rho != 32) return TRI_EINVAL;
    size_t need = 0;
    switch (mode) {
        case TRI_DUMMY_FIXED: need = 4; break;
        case TRI_DUMMY_PACKED:
            if (!map->diag || (map->world > 1 && !map->snap)) return TRI_EINVAL;
            need = map->out_cells * (map->n <= 65536 ? 4u : 8u);
            break;
        case TRI_DUMMY_DIGEST: need = 8; break;
        case TRI_DUMMY_COUNT: need = 5 * 8; break;
        default: return TRI_EINVAL;
    }
    if (out_bytes < need) return TRI_EINVAL;
    if (strategy == TRI_RB) return launch_dummy_rb(*map, mode, d_out, (cudaStream_t)stream);
    return launch_dummy(*map, strategy, mode, d_out, (cudaStream_t)stream);
}

extern "C++" {
namespace tri {
// Validation shared by tri_edm and tri_edm_host (include/tri.h): the map, the
// strategy, the tile edge, the point layout and both capacities.
bool edm_args_bad(const tri_map_t *map, int32_t strategy, int32_t dim, int64_t ld, size_t pts_bytes,
                  size_t out_bytes) {
    if (bad_map(map) || (bad_strategy(strategy) && strategy != TRI_RB && strategy != TRI_LAMBDA_CLC)) return true;
    if (!map->diag || (map->world > 1 && !map->snap)) return true;
    if (strategy == TRI_RB && map->world != 1) return true;
    if (map->rho != 32 && map->rho != 64 && map->rho != 128 && map->rho != 256) return true;
    if (dim < 1 || dim > 4 || ld < dim || ld > (1ll << 20)) return true;
    const uint64_t need_pts = 4ull * ((uint64_t)(map->n - 1) * (uint64_t)ld + (uint64_t)dim);
    if (pts_bytes < need_pts) return true;
    if (out_bytes / 4u < map->out_cells) return true;
    return false;
}
}  // namespace tri
}  // extern "C++"

tri_status tri_edm(const tri_map_t *map, int32_t strategy, const float *d_pts, int32_t dim, int64_t ld,
                   size_t pts_bytes, float *d_out, size_t out_bytes, void *stream) {
    g_launches = 0;
    if (!d_pts || !d_out || edm_args_bad(map, strategy, dim, ld, pts_bytes, out_bytes)) return TRI_EINVAL;
    if (((uintptr_t)d_out & (map->rho == 256 ? 31u : 15u)) != 0) return TRI_EINVAL;   // 32-B chunks at rho 256
    if (map->out_cells == 0) return TRI_OK;
    if (strategy == TRI_RB) return launch_edm_rb(*map, d_pts, dim, ld, d_out, (cudaStream_t)stream);
    return launch_edm(*map, strategy, d_pts, dim, ld, d_out, (cudaStream_t)stream);
}

size_t tri_collide_workspace_size(const tri_map_t *map, int32_t strategy) {
    if (bad_map(map)) return 0;
    return (strategy == TRI_LAMBDA_TC || strategy == TRI_BB_TC) ? collide_tc_ws_bytes(*map) : 0;
}

tri_status tri_tc_tf32_probe(const float *d_x, const float *d_y, float *d_d, void *stream) {
    g_launches = 0;
    if (!d_x || !d_y || !d_d) return TRI_EINVAL;
    return launch_tc_tf32_probe(d_x, d_y, d_d, (cudaStream_t)stream);
}

tri_status tri_tc_f16_probe(const void *d_x, const void *d_y, void *d_d, void *stream) {
    g_launches = 0;
    if (!d_x || !d_y || !d_d) return TRI_EINVAL;
    return launch_tc_f16_probe(d_x, d_y, d_d, (cudaStream_t)stream);
}

tri_status tri_collide(const tri_map_t *map, int32_t strategy, const float *d_spheres, size_t spheres_bytes,
                       unsigned long long *d_count, size_t count_bytes, void *d_ws, size_t ws_bytes,
                       void *stream) {
    g_launches = 0;
    const bool tc = strategy == TRI_LAMBDA_TC || strategy == TRI_BB_TC;
    if (bad_map(map) || (bad_strategy(strategy) && !tc) || !d_spheres || !d_count) return TRI_EINVAL;
    if (tc ? (map->rho % 128 || map->rho < 256 || map->rho > 1024)     // tcgen05: 256, 384, ..., 1024
           : (map->rho != 128 && map->rho != 256 && map->rho != 512))
        return TRI_EINVAL;
    if (((uintptr_t)d_spheres & 15u) != 0 || (((uintptr_t)d_count) & 7u)) return TRI_EINVAL;
    if (spheres_bytes / 16u < (uint64_t)map->n || count_bytes < 8) return TRI_EINVAL;
    if (tc) {
        if (!d_ws || ws_bytes < collide_tc_ws_bytes(*map) || (((uintptr_t)d_ws) & 15u)) return TRI_EINVAL;
        if (map->rho == 128) return TRI_EINVAL;
        return launch_collide_tc(*map, strategy, d_spheres, d_count, d_ws, (cudaStream_t)stream);
    }
    return launch_collide(*map, strategy, d_spheres, d_count, (cudaStream_t)stream);
}

size_t tri_ca_workspace_size(const tri_map_t *map) {
    (void)map;
    return 0;
}

// Capacities of a CA call: state slices and the k-row halos (include/tri.h).
static bool ca_bytes_bad(const tri_map_t *m, int32_t k, size_t in_bytes, size_t out_bytes, const void *above,
                         size_t above_bytes, const void *below, size_t below_bytes) {
    if (in_bytes < m->out_cells || out_bytes < m->out_cells) return true;
    const uint64_t rb = (uint64_t)m->row_begin, re = (uint64_t)m->row_end, n = (uint64_t)m->n;
    const uint64_t lo = rb > (uint64_t)k ? rb - (uint64_t)k : 0, hi = re + (uint64_t)k < n ? re + (uint64_t)k : n;
    if (above && rb > 0 && above_bytes < T2(rb) - T2(lo)) return true;
    if (below && re < n && below_bytes < T2(hi) - T2(re)) return true;
    return false;
}

tri_status tri_ca_step(const tri_map_t *map, int32_t strategy, const uint8_t *d_in, size_t in_bytes,
                       uint8_t *d_out, size_t out_bytes, const uint8_t *d_halo_above, size_t above_bytes,
                       const uint8_t *d_halo_below, size_t below_bytes, void *d_ws, void *stream) {
    g_launches = 0;
    (void)d_ws;
    if (bad_map(map) || bad_strategy(strategy) || !d_in || !d_out || d_in == d_out) return TRI_EINVAL;
    if (ca_bytes_bad(map, 1, in_bytes, out_bytes, d_halo_above, above_bytes, d_halo_below, below_bytes))
        return TRI_EINVAL;
    if (!map->diag || (map->world > 1 && !map->snap)) return TRI_EINVAL;
    if (map->rho != 128 && map->rho != 224 && map->rho != 256 && map->rho != 512) return TRI_EINVAL;
    if ((((uintptr_t)d_in) | ((uintptr_t)d_out)) & 15u) return TRI_EINVAL;
    if (map->out_cells == 0) return TRI_OK;
    return launch_ca(*map, strategy, d_in, d_out, d_halo_above, d_halo_below, (cudaStream_t)stream);
}

tri_status tri_ca_steps(const tri_map_t *map, int32_t strategy, int32_t k, const uint8_t *d_in, size_t in_bytes,
                        uint8_t *d_out, size_t out_bytes, const uint8_t *d_halo_above, size_t above_bytes,
                        const uint8_t *d_halo_below, size_t below_bytes, void *d_ws, void *stream) {
    g_launches = 0;
    (void)d_ws;
    if (bad_map(map) || bad_strategy(strategy) || !d_in || !d_out || d_in == d_out) return TRI_EINVAL;
    if (!map->diag || (map->world > 1 && !map->snap)) return TRI_EINVAL;
    if (k < 1 || !((map->rho == 128 && k <= 16) || (map->rho == 224 && k <= 8))) return TRI_EINVAL;
    if (ca_bytes_bad(map, k, in_bytes, out_bytes, d_halo_above, above_bytes, d_halo_below, below_bytes))
        return TRI_EINVAL;
    if ((((uintptr_t)d_in) | ((uintptr_t)d_out)) & 15u) return TRI_EINVAL;
    if (map->out_cells == 0) return TRI_OK;
    return launch_ca_steps(*map, strategy, k, d_in, d_out, d_halo_above, d_halo_below, nullptr, nullptr,
                           (cudaStream_t)stream);
}

tri_status tri_ca_steps_p2p(const tri_map_t *map, int32_t strategy, int32_t k, const uint8_t *d_in,
                            size_t in_bytes, uint8_t *d_out, size_t out_bytes, const uint8_t *d_halo_above,
                            size_t above_bytes, const uint8_t *d_halo_below, size_t below_bytes,
                            uint8_t *d_peer_above, uint8_t *d_peer_below, void *d_ws, void *stream) {
    g_launches = 0;
    (void)d_ws;
    if (bad_map(map) || bad_strategy(strategy) || !d_in || !d_out || d_in == d_out) return TRI_EINVAL;
    if (!map->diag || (map->world > 1 && !map->snap)) return TRI_EINVAL;
    if (k < 1 || !((map->rho == 128 && k <= 16) || (map->rho == 224 && k <= 8))) return TRI_EINVAL;
    if (ca_bytes_bad(map, k, in_bytes, out_bytes, d_halo_above, above_bytes, d_halo_below, below_bytes))
        return TRI_EINVAL;
    if ((((uintptr_t)d_in) | ((uintptr_t)d_out) | ((uintptr_t)d_peer_above) | ((uintptr_t)d_peer_below)) & 15u)
        return TRI_EINVAL;
    // every peer row this rank sends must be its own: it owns >= k rows (or none)
    if ((d_peer_above || d_peer_below) && map->row_end > map->row_begin && map->row_end - map->row_begin < k)
        return TRI_EINVAL;
    if (map->out_cells == 0) return TRI_OK;
    return launch_ca_steps(*map, strategy, k, d_in, d_out, d_halo_above, d_halo_below, d_peer_above, d_peer_below,
                           (cudaStream_t)stream);
}

size_t tri_ca_run_workspace_size(const tri_map_t *map) {
    if (bad_map(map)) return 0;
    return ca_run_ws_bytes(*map);
}

tri_status tri_ca_run(const tri_map_t *map, int32_t strategy, int64_t steps, const uint8_t *d_in, size_t in_bytes,
                      uint8_t *d_out, size_t out_bytes, void *d_ws, size_t ws_bytes, void *stream) {
    g_launches = 0;
    if (bad_map(map) || bad_strategy(strategy) || !d_in || !d_out || !d_ws || steps < 0) return TRI_EINVAL;
    if (!map->diag || map->world != 1 || map->rho != 240) return TRI_EINVAL;
    if (in_bytes < map->cells || out_bytes < map->cells || ws_bytes < ca_run_ws_bytes(*map)) return TRI_EINVAL;
    if ((((uintptr_t)d_in) | ((uintptr_t)d_out) | ((uintptr_t)d_ws)) & 15u) return TRI_EINVAL;
    if (strategy == TRI_BB && map->m > 65535) return TRI_EINVAL;
    return launch_ca_run(*map, strategy, steps, d_in, d_out, d_ws, (cudaStream_t)stream);
}

tri_status tri_ipc_handle(const void *d_ptr, void *handle, uint64_t *offset) {
    if (!d_ptr || !handle || !offset) return TRI_EINVAL;
    void *base = nullptr;
    size_t size = 0;
    if (cuda_driver_range(d_ptr, &base, &size) != TRI_OK) return TRI_ECUDA;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, base) != cudaSuccess) return TRI_ECUDA;
    static_assert(sizeof(h) == TRI_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &h, sizeof(h));
    *offset = (uint64_t)((const char *)d_ptr - (const char *)base);
    return TRI_OK;
}

tri_status tri_ipc_open(const void *handle, uint64_t offset, void **d_ptr, void **d_base) {
    if (!handle || !d_ptr || !d_base) return TRI_EINVAL;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void *base = nullptr;
    if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return TRI_ECUDA;
    *d_base = base;
    *d_ptr = (char *)base + offset;
    return TRI_OK;
}

tri_status tri_ipc_close(void *d_base) {
    if (!d_base) return TRI_EINVAL;
    return cudaIpcCloseMemHandle(d_base) == cudaSuccess ? TRI_OK : TRI_ECUDA;
}

tri_status tet_map_init(tet_map_t *map, int64_t n, int32_t rho, int32_t rank, int32_t world) {
    if (!map || n < 3 || (rho != 4 && rho != 8 && rho != 16 && rho != 32) || world < 1 || rank < 0 ||
        rank >= world)
        return TRI_EINVAL;
    if (n > (1ll << 22)) return TRI_ERANGE;
    tet_map_t t;
    std::memset(&t, 0, sizeof t);
    t.n = n; t.rho = rho; t.rank = rank; t.world = world;
    t.m = (n + rho - 1) / rho;
    const uint64_t m = (uint64_t)t.m;
    t.blocks = T3(m);
    if (t.blocks >= TRI_OMEGA_MAX) return TRI_ERANGE;
    t.omega_begin = (uint64_t)(((unsigned __int128)rank * t.blocks) / (uint64_t)world);
    t.omega_end = (uint64_t)(((unsigned __int128)(rank + 1) * t.blocks) / (uint64_t)world);
    const uint64_t r3 = (uint64_t)rho * rho * rho;
    const uint64_t nn = (uint64_t)n;
    const uint64_t useful = nn * (nn - 1) * (nn - 2) / 6;   // C(n,3): p > q > s
    t.waste_tet = t.blocks * r3 - useful;
    t.waste_bb = m * m * m * r3 - useful;
    *map = t;
    return TRI_OK;
}

tri_status tet_lambda(uint64_t omega, uint32_t *i, uint32_t *j, uint32_t *k) {
    if (!i || !j || !k) return TRI_EINVAL;
    if (omega >= TRI_OMEGA_MAX) return TRI_ERANGE;
    tet_map(omega, *i, *j, *k);
    return TRI_OK;
}

tri_status tet_map_eval(uint64_t omega0, uint64_t count, uint32_t *d_ijk, unsigned long long *d_fail,
                        void *stream) {
    g_launches = 0;
    if (!d_fail) return TRI_EINVAL;
    if (omega0 > TRI_OMEGA_MAX || count > TRI_OMEGA_MAX - omega0) return TRI_ERANGE;
    if (d_ijk && count >= (1ull << 30)) return TRI_EINVAL;
    return launch_tet_map_eval(omega0, count, d_ijk, d_fail, (cudaStream_t)stream);
}

size_t tet_lut_bytes(uint32_t kmax, int32_t shift) {
    if (kmax == 0 || kmax >= (1u << 20) || shift < 0 || shift > 40) return 0;
    const uint64_t nb = (T3((uint64_t)kmax + 1) >> shift) + 1;
    return (size_t)(8ull * ((uint64_t)kmax + 2) + 4ull * (nb + 1));
}

tri_status tet_lut_build(uint32_t kmax, int32_t shift, void *d_lut, size_t lut_bytes, void *stream) {
    g_launches = 0;
    const size_t need = tet_lut_bytes(kmax, shift);
    if (!need || !d_lut || lut_bytes < need || ((uintptr_t)d_lut & 7u)) return TRI_EINVAL;
    return launch_tet_lut_build(kmax, shift, d_lut, (cudaStream_t)stream);
}

tri_status tet_map_eval_lut(uint64_t omega0, uint64_t count, uint32_t kmax, int32_t shift, const void *d_lut,
                            uint32_t *d_ijk, unsigned long long *d_fail, void *stream) {
    g_launches = 0;
    if (!d_fail || !d_lut || !tet_lut_bytes(kmax, shift) || ((uintptr_t)d_lut & 7u)) return TRI_EINVAL;
    if (d_ijk && count >= (1ull << 30)) return TRI_EINVAL;
    const uint64_t end = T3((uint64_t)kmax + 1);              // omega + 1 is mapped too
    if (omega0 >= end || count > end - 1 - omega0) return TRI_ERANGE;
    return launch_tet_map_eval_lut(omega0, count, kmax, shift, d_lut, d_ijk, d_fail, (cudaStream_t)stream);
}

tri_status tet_triplet(const tet_map_t *map, int32_t strategy, const float *d_pts4, size_t pts_bytes, double nu,
                       double *d_energy, size_t energy_bytes, void *stream) {
    g_launches = 0;
    if (!map || bad_strategy(strategy) || !d_pts4 || !d_energy) return TRI_EINVAL;
    if (map->n < 3 || pts_bytes / 16u < (uint64_t)map->n || energy_bytes / 8u < (uint64_t)map->n ||
        (((uintptr_t)d_energy) & 7u))
        return TRI_EINVAL;
    if (map->n < 3 || map->m != (map->n + map->rho - 1) / map->rho || map->blocks != T3((uint64_t)map->m) ||
        map->omega_end > map->blocks || map->omega_begin > map->omega_end)
        return TRI_EINVAL;
    if (((uintptr_t)d_pts4 & 15u) != 0) return TRI_EINVAL;
    return launch_triplet(*map, strategy, d_pts4, nu, d_energy, (cudaStream_t)stream);
}

int32_t tri_last_launch_count(void) { return g_launches; }

const char *tri_status_str(tri_status s) {
    switch (s) {
        case TRI_OK: return "TRI_OK";
        case TRI_EINVAL: return "TRI_EINVAL: invalid argument";
        case TRI_ERANGE: return "TRI_ERANGE: size exceeds the 64-bit / 2^40 bound";
        case TRI_ECUDA: return "TRI_ECUDA: CUDA error";
        case TRI_ENOTSUP: return "TRI_ENOTSUP: not supported";
    }
    return "unknown tri_status";
}

}  // extern "C"
