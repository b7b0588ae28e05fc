// gather.cu -- mini-batch row gather (K7): Fig. 2 step 2 "lookup the memory and
// the mailbox for the supporting nodes", plus edge features by eid (Table 3: random
// 128-d edge features for LastFM).  out_t[i] = table_t[ids[i]] byte for byte.
//
// HBM-bound byte copy: each thread moves one 16-B (or 8/4/2/1-B, by alignment) chunk of a row;
// the flat (row, chunk) index space makes consecutive lanes touch consecutive bytes of a row, so
// every row read and every output write is a full-sector, coalesced transfer.  kUnroll
// independent chunks per thread are loaded before any is stored (memory-level parallelism).
// One persistent launch covers all tables; the id count may be a device scalar written by the
// sampler (no host sync between tgl_sample and tgl_gather).
#include <algorithm>

#include "common.cuh"

namespace tgl {

__device__ int g_gather_err = 0;  // sticky error word of tgl_gather (read by tgl_check(NULL))

struct GatherTable {
    const unsigned char* table;
    unsigned char* out;
    int64_t n_rows;
    int64_t row_bytes;
    uint32_t vec_shift;        // log2 of the chunk width
    uint32_t chunks_per_row;   // row_bytes >> vec_shift
};

struct GatherParams {
    const int32_t* ids;
    int64_t n_cap;
    const int64_t* n_dev;
    int32_t n_tables;
    GatherTable t[TGL_MAX_GATHER_TABLES];
};

constexpr int kGatherThreads = 256;
constexpr int kUnroll = 4;

template <int VS>
__device__ __forceinline__ void gather_table(const int32_t* __restrict__ ids, int64_t n, const GatherTable& g,
                                             int* bad) {
    using T = typename Vec<VS>::T;
    const uint64_t cpr = g.chunks_per_row;
    const uint64_t total = (uint64_t)n * cpr;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const T* __restrict__ src = reinterpret_cast<const T*>(g.table);
    T* __restrict__ dst = reinterpret_cast<T*>(g.out);
    for (uint64_t e0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < total; e0 += stride * kUnroll) {
        T v[kUnroll];
        uint64_t e[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            e[u] = e0 + (uint64_t)u * stride;
            T x;
            memset(&x, 0, sizeof(T));
            if (e[u] < total) {
                const uint64_t row = cpr == 1 ? e[u] : e[u] / cpr;
                const uint64_t c = e[u] - row * cpr;
                const int64_t id = __ldg(ids + row);
                if ((uint64_t)id < (uint64_t)g.n_rows)
                    x = __ldg(src + (uint64_t)id * cpr + c);
                else if (id != -1 && c == 0)
                    *bad = 1;
            }
            v[u] = x;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (e[u] < total) __stcs(dst + e[u], v[u]);
    }
}

__global__ void __launch_bounds__(kGatherThreads) gather_kernel(const __grid_constant__ GatherParams p) {
    int64_t n = p.n_cap;
    if (p.n_dev) {
        const int64_t m = *p.n_dev;
        n = m < n ? (m > 0 ? m : 0) : n;
    }
    int bad = 0;
    for (int j = 0; j < p.n_tables; ++j) {
        const GatherTable& g = p.t[j];
        switch (g.vec_shift) {
            case 4: gather_table<4>(p.ids, n, g, &bad); break;
            case 3: gather_table<3>(p.ids, n, g, &bad); break;
            case 2: gather_table<2>(p.ids, n, g, &bad); break;
            case 1: gather_table<1>(p.ids, n, g, &bad); break;
            default: gather_table<0>(p.ids, n, g, &bad); break;
        }
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(&g_gather_err, kErrRange);
}

int read_and_clear_gather_err(cudaStream_t st, int* bits) {
    int* dptr = nullptr;
    if (cudaGetSymbolAddress((void**)&dptr, g_gather_err) != cudaSuccess) return TGL_ECUDA;
    if (cudaMemcpyAsync(bits, dptr, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess) return TGL_ECUDA;
    if (cudaMemsetAsync(dptr, 0, sizeof(int), st) != cudaSuccess) return TGL_ECUDA;
    return TGL_OK;
}

}  // namespace tgl

using namespace tgl;

extern "C" int tgl_gather(const int32_t* ids, int64_t n_ids_cap, const int64_t* n_ids_dev,
                          const tgl_gather_table* tables, int32_t n_tables, void* stream) {
    NvtxRange nvtx_("tgl_gather");
    if (n_tables < 0 || n_tables > TGL_MAX_GATHER_TABLES || n_ids_cap < 0) return TGL_EINVAL;
    if (n_tables > 0 && !tables) return TGL_EINVAL;
    if (n_ids_cap > 0 && !ids) return TGL_EINVAL;
    int rc = check_device();
    if (rc) return rc;
    GatherParams gp;
    memset(&gp, 0, sizeof(gp));
    gp.ids = ids;
    gp.n_cap = n_ids_cap;
    gp.n_dev = n_ids_dev;
    gp.n_tables = n_tables;
    uint64_t max_work = 0;
    for (int j = 0; j < n_tables; ++j) {
        const tgl_gather_table& t = tables[j];
        if (t.row_bytes <= 0 || t.n_rows < 0) return TGL_EINVAL;
        if ((t.n_rows > 0 && !t.table) || (n_ids_cap > 0 && !t.out)) return TGL_EINVAL;
        const uintptr_t align = (uintptr_t)t.table | (uintptr_t)t.out | (uintptr_t)t.row_bytes;
        uint32_t vs = 4;
        while (vs > 0 && (align & ((1u << vs) - 1))) --vs;
        if ((uint64_t)(t.row_bytes >> vs) >= (1ull << 32)) return TGL_EINVAL;
        GatherTable& g = gp.t[j];
        g.table = static_cast<const unsigned char*>(t.table);
        g.out = static_cast<unsigned char*>(t.out);
        g.n_rows = t.n_rows;
        g.row_bytes = t.row_bytes;
        g.vec_shift = vs;
        g.chunks_per_row = (uint32_t)(t.row_bytes >> vs);
        max_work = std::max<uint64_t>(max_work, (uint64_t)n_ids_cap * g.chunks_per_row);
    }
    if (n_tables == 0 || n_ids_cap == 0) return TGL_OK;
    const uint64_t per_cta = (uint64_t)kGatherThreads * kUnroll;
    const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>((max_work + per_cta - 1) / per_cta, 148ull * 8));
    gather_kernel<<<(unsigned)grid, kGatherThreads, 0, (cudaStream_t)stream>>>(gp);
    return cudaGetLastError() == cudaSuccess ? TGL_OK : TGL_ECUDA;
}
