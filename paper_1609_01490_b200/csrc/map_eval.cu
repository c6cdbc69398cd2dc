// map_eval.cu -- GPU self-check of the 2-D and tetrahedral maps.
//
// For every omega in [w0, w0+count) the kernel evaluates the production map
// (tri::lambda_map / tri::tet_map, the exact functions the workload kernels
// use) and counts violations of
//   Eq. 3:        T(i) <= omega < T(i+1), j <= i
//   Eq. 1 successor: lambda(omega+1) in {(i, j+1), (i+1, 0)}
// and for the tetrahedron the layer property T3(k) <= omega < T3(k+1),
// j <= i <= k, and the layer-major successor rule.  A persistent grid walks
// the range with a stride; each lane carries its own omega (no shuffles), and
// failure counts are reduced per warp before one atomic.
#include "tri_common.cuh"

namespace {

__global__ void __launch_bounds__(256) map_eval_kernel(uint64_t w0, uint64_t count, uint32_t *ij,
                                                       unsigned long long *fail) {
    unsigned long long bad = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) {
        const uint64_t w = w0 + t;
        uint32_t i, j;
        tri::lambda_map(w, i, j);
        const uint64_t Ti = tri::T2(i);
        bool ok = (Ti <= w) && (w < Ti + i + 1) && (j <= i) && (Ti + j == w);
        uint32_t i2, j2;
        tri::lambda_map(w + 1, i2, j2);
        ok = ok && ((i2 == i && j2 == j + 1) || (i2 == i + 1 && j2 == 0));
        bad += ok ? 0 : 1;
        if (ij) { ij[2 * t] = i; ij[2 * t + 1] = j; }
    }
    bad = __reduce_add_sync(0xffffffffu, (unsigned)bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(fail, bad);
}

__global__ void __launch_bounds__(256) tet_eval_kernel(uint64_t w0, uint64_t count, uint32_t *ijk,
                                                       unsigned long long *fail) {
    unsigned long long bad = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) {
        const uint64_t w = w0 + t;
        uint32_t i, j, k;
        tri::tet_map(w, i, j, k);
        const uint64_t Tk = tri::T3(k);
        bool ok = (Tk <= w) && (w < tri::T3((uint64_t)k + 1)) && (j <= i) && (i <= k) &&
                  (Tk + tri::T2(i) + j == w);
        uint32_t i2, j2, k2;
        tri::tet_map(w + 1, i2, j2, k2);
        ok = ok && ((k2 == k && i2 == i && j2 == j + 1) || (k2 == k && i2 == i + 1 && j2 == 0) ||
                    (k2 == k + 1 && i2 == 0 && j2 == 0));
        bad += ok ? 0 : 1;
        if (ijk) { ijk[3 * t] = i; ijk[3 * t + 1] = j; ijk[3 * t + 2] = k; }
    }
    bad = __reduce_add_sync(0xffffffffu, (unsigned)bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(fail, bad);
}

// Validity scan of a square-root variant (section 4.1): compare the uncorrected
// variant with the exact map; count mismatches and keep the first failing omega.
__global__ void __launch_bounds__(256) variant_scan_kernel(int variant, uint64_t w0, uint64_t count,
                                                           unsigned long long *fail, unsigned long long *first) {
    unsigned long long bad = 0, mine = ~0ull;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) {
        const uint64_t w = w0 + t;
        uint32_t i, j, vi, vj;
        tri::lambda_map(w, i, j);
        tri::lambda_variant(w, variant, vi, vj);
        if (vi != i || vj != j) {
            ++bad;
            if (w < mine) mine = w;
        }
    }
    bad = __reduce_add_sync(0xffffffffu, (unsigned)bad);
    for (int o = 16; o; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, mine, o);
        mine = other < mine ? other : mine;
    }
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicAdd(fail, bad);
        if (mine != ~0ull) atomicMin(first, mine);
    }
}

// Rows of an uncorrected square-root variant: rows[t] = the variant's i at omega0 + t.
__global__ void __launch_bounds__(256) variant_rows_kernel(int variant, uint64_t w0, uint64_t count, uint32_t *rows) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) {
        uint32_t vi, vj;
        tri::lambda_variant(w0 + t, variant, vi, vj);
        rows[t] = vi;
    }
}

// ---- succinct layer table: S[k] = T3(k), G[g] = max{k : T3(k) <= g << shift}
struct TetLut {
    const uint64_t *S;
    const uint32_t *G;
    int shift;
};

__host__ __device__ __forceinline__ TetLut lut_view(const void *d, uint32_t kmax, int shift) {
    TetLut L;
    L.S = (const uint64_t *)d;
    L.G = (const uint32_t *)(L.S + (uint64_t)kmax + 2);
    L.shift = shift;
    return L;
}

// layer k from the table: bisection over [G[g], G[g+1]] on S (no cube root)
__device__ __forceinline__ void tet_map_lut(const TetLut &L, uint64_t w, uint32_t &i, uint32_t &j, uint32_t &k) {
    const uint64_t g = w >> L.shift;
    uint32_t lo = __ldg(L.G + g), hi = __ldg(L.G + g + 1);
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (__ldg(L.S + mid) <= w) lo = mid;
        else hi = mid - 1;
    }
    k = lo;
    tri::lambda_map(w - __ldg(L.S + lo), i, j);
}

__global__ void __launch_bounds__(256) tet_lut_build_kernel(uint32_t kmax, int shift, uint64_t *S, uint32_t *G,
                                                            uint64_t nb) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= (uint64_t)kmax + 1; t += stride)
        S[t] = tri::T3(t);
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g <= nb; g += stride) {
        const uint64_t w = g << shift;
        uint32_t lo = 0, hi = kmax + 1;                       // largest k <= kmax + 1 with T3(k) <= w
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (tri::T3(mid) <= w) lo = mid;
            else hi = mid - 1;
        }
        G[g] = lo;
    }
}

__global__ void __launch_bounds__(256) tet_eval_lut_kernel(uint64_t w0, uint64_t count, TetLut L, uint32_t *ijk,
                                                           unsigned long long *fail) {
    unsigned long long bad = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) {
        const uint64_t w = w0 + t;
        uint32_t i, j, k;
        tet_map_lut(L, w, i, j, k);
        const uint64_t Tk = tri::T3(k);
        bool ok = (Tk <= w) && (w < tri::T3((uint64_t)k + 1)) && (j <= i) && (i <= k) &&
                  (Tk + tri::T2(i) + j == w);
        uint32_t i2, j2, k2;
        tet_map_lut(L, w + 1, i2, j2, k2);
        ok = ok && ((k2 == k && i2 == i && j2 == j + 1) || (k2 == k && i2 == i + 1 && j2 == 0) ||
                    (k2 == k + 1 && i2 == 0 && j2 == 0));
        bad += ok ? 0 : 1;
        if (ijk) { ijk[3 * t] = i; ijk[3 * t + 1] = j; ijk[3 * t + 2] = k; }
    }
    bad = __reduce_add_sync(0xffffffffu, (unsigned)bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(fail, bad);
}

unsigned eval_grid(uint64_t count) {
    uint64_t want = (count + 255) / 256;
    uint64_t cap = (uint64_t)tri::sm_count() * 8ull * 16ull;
    if (want > cap) want = cap;
    return (unsigned)(want ? want : 1);
}

}  // namespace

namespace tri {

tri_status launch_map_eval(uint64_t w0, uint64_t count, uint32_t *d_ij, unsigned long long *d_fail,
                           cudaStream_t st) {
    if (cudaMemsetAsync(d_fail, 0, sizeof(unsigned long long), st) != cudaSuccess) return TRI_ECUDA;
    if (count == 0) return TRI_OK;
    map_eval_kernel<<<eval_grid(count), 256, 0, st>>>(w0, count, d_ij, d_fail);
    note_launches(1);
    return cuda_status();
}

tri_status launch_variant_scan(int variant, uint64_t w0, uint64_t count, unsigned long long *d_fail,
                               unsigned long long *d_first, cudaStream_t st) {
    if (cudaMemsetAsync(d_fail, 0, sizeof(unsigned long long), st) != cudaSuccess) return TRI_ECUDA;
    if (cudaMemsetAsync(d_first, 0xff, sizeof(unsigned long long), st) != cudaSuccess) return TRI_ECUDA;
    if (count == 0) return TRI_OK;
    variant_scan_kernel<<<eval_grid(count), 256, 0, st>>>(variant, w0, count, d_fail, d_first);
    note_launches(1);
    return cuda_status();
}

tri_status launch_variant_rows(int variant, uint64_t w0, uint64_t count, uint32_t *d_rows, cudaStream_t st) {
    if (count == 0) return TRI_OK;
    variant_rows_kernel<<<eval_grid(count), 256, 0, st>>>(variant, w0, count, d_rows);
    note_launches(1);
    return cuda_status();
}

tri_status launch_tet_map_eval(uint64_t w0, uint64_t count, uint32_t *d_ijk, unsigned long long *d_fail,
                               cudaStream_t st) {
    if (cudaMemsetAsync(d_fail, 0, sizeof(unsigned long long), st) != cudaSuccess) return TRI_ECUDA;
    if (count == 0) return TRI_OK;
    tet_eval_kernel<<<eval_grid(count), 256, 0, st>>>(w0, count, d_ijk, d_fail);
    note_launches(1);
    return cuda_status();
}

tri_status launch_tet_lut_build(uint32_t kmax, int shift, void *d_lut, cudaStream_t st) {
    uint64_t *S = (uint64_t *)d_lut;
    uint32_t *G = (uint32_t *)(S + (uint64_t)kmax + 2);
    const uint64_t nb = (T3((uint64_t)kmax + 1) >> shift) + 1;
    const uint64_t n = nb > (uint64_t)kmax + 2 ? nb : (uint64_t)kmax + 2;
    tet_lut_build_kernel<<<eval_grid(n), 256, 0, st>>>(kmax, shift, S, G, nb);
    note_launches(1);
    return cuda_status();
}

tri_status launch_tet_map_eval_lut(uint64_t w0, uint64_t count, uint32_t kmax, int shift, const void *d_lut,
                                   uint32_t *d_ijk, unsigned long long *d_fail, cudaStream_t st) {
    if (cudaMemsetAsync(d_fail, 0, sizeof(unsigned long long), st) != cudaSuccess) return TRI_ECUDA;
    if (count == 0) return TRI_OK;
    tet_eval_lut_kernel<<<eval_grid(count), 256, 0, st>>>(w0, count, lut_view(d_lut, kmax, shift), d_ijk, d_fail);
    note_launches(1);
    return cuda_status();
}

}  // namespace tri
