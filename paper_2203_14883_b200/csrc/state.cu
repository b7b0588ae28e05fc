// state.cu -- the state write of Fig. 2 step 6 ("update the memory and the mailbox
// for next mini-batch"; L210 the mailbox keeps "a fixed number of most recent mails"; L322 1 mail,
// 10 for APAN).  Semantics (R#25): events i = 0..n-1 are applied in batch order; event i
// of node v writes its row(s) into slot pos[v] of v's K-slot ring, then pos[v] = (pos[v]+1) mod K.
// K = 1 is "the last event of v wins" (node memory, mem_ts, the 1-mail mailbox).
//
// The sequential definition is parallelised without any order-dependent atomics:
//   S1 state_keys_kernel    key = node id (out-of-range: sentinel n_nodes, sticky ERANGE)
//   S2 radix passes          stable LSD sort of (key, event index) by key (radix.cuh): a node's
//                            events become one contiguous run, still in batch order
//   S3 state_slot_kernel     per sorted position j of node v: run [first, first + m) by two binary
//                            searches over the sorted keys; q = j - first.  Only the last K events
//                            of the run survive (earlier ones would be overwritten in the ring):
//                            slot = (pos[v] + q) mod K, destination row v*K + slot (distinct per
//                            survivor, so the result is deterministic); ts_table written here
//   S4 state_copy_kernel     flat (survivor, 16-B chunk) scatter of every table's row, the same
//                            index space as tgl_gather (coalesced row reads and writes)
//   S5 state_cursor_kernel   run tails advance pos[v] by m mod K (after S3 has read it)
#include <algorithm>

#include "common.cuh"
#include "radix.cuh"
#include "scan.cuh"

namespace tgl {

__device__ int g_state_err = 0;  // sticky error word of tgl_state_write (read by tgl_check(NULL))

struct StateTable {
    const unsigned char* rows;
    unsigned char* table;
    uint32_t vec_shift;
    uint32_t chunks_per_row;
};

struct StateParams {
    const uint32_t* keys;  // sorted node ids (sentinel n_nodes for bad ids)
    const uint32_t* evt;   // event index of sorted position j
    const int64_t* dst;    // destination row (v*K + slot) of sorted position j, or -1
    int64_t n;
    int32_t n_tables;
    StateTable t[TGL_MAX_GATHER_TABLES];
};

__global__ void state_keys_kernel(const int32_t* __restrict__ ids, int64_t n, int32_t n_nodes,
                                  uint32_t* __restrict__ keys) {
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i - (threadIdx.x & 31) < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n) {
            const int32_t v = ids[i];
            const bool ok = (uint32_t)v < (uint32_t)n_nodes;
            keys[i] = ok ? (uint32_t)v : (uint32_t)n_nodes;
            bad |= !ok;
        }
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(&g_state_err, kErrRange);
}

__device__ __forceinline__ int64_t first_geq(const uint32_t* keys, int64_t n, uint32_t v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(keys + mid) < v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__global__ void state_slot_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ evt, int64_t n,
                                  int32_t n_nodes, int32_t K, const int32_t* __restrict__ pos,
                                  const float* __restrict__ ts, float* __restrict__ ts_table,
                                  int64_t* __restrict__ dst) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = keys[j];
        int64_t d = -1;
        if (v < (uint32_t)n_nodes) {
            const int64_t first = first_geq(keys, n, v);
            const int64_t m = first_geq(keys, n, v + 1) - first;
            const int64_t q = j - first;
            if (q + K >= m) {  // among the last K events of the run
                const int64_t base = (K > 1 && pos) ? (int64_t)pos[v] : 0;
                d = (int64_t)v * K + (base + q) % K;
                if (ts_table) ts_table[d] = ts[evt[j]];
            }
        }
        dst[j] = d;
    }
}

// Rows to warps: a warp copies R = max(1, 32 / cpr) rows at a time, lane = (row, chunk); rows of
// more than 32 chunks are strided over the lanes.  Row reads and table writes are contiguous.
template <int VS>
__device__ __forceinline__ void state_copy_table(const StateParams& p, const StateTable& t) {
    using T = typename Vec<VS>::T;
    const uint32_t cpr = t.chunks_per_row;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t R = cpr >= 32 ? 1u : 32u / cpr;
    const uint32_t sub = cpr >= 32 ? 0u : lane / cpr;
    const uint32_t c0 = lane - sub * (cpr >= 32 ? 0u : cpr);
    const T* __restrict__ src = reinterpret_cast<const T*>(t.rows);
    T* __restrict__ out = reinterpret_cast<T*>(t.table);
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (sub >= R) return;
    for (int64_t j = warp * R + sub; j < p.n; j += n_warps * R) {
        const int64_t d = __ldg(p.dst + j);
        if (d < 0) continue;
        const T* s = src + (uint64_t)__ldg(p.evt + j) * cpr;
        T* o = out + (uint64_t)d * cpr;
        for (uint32_t c = c0; c < cpr; c += 32) o[c] = __ldg(s + c);
    }
}

__global__ void __launch_bounds__(256) state_copy_kernel(const __grid_constant__ StateParams p) {
    for (int j = 0; j < p.n_tables; ++j) {
        const StateTable& t = p.t[j];
        switch (t.vec_shift) {
            case 4: state_copy_table<4>(p, t); break;
            case 3: state_copy_table<3>(p, t); break;
            case 2: state_copy_table<2>(p, t); break;
            case 1: state_copy_table<1>(p, t); break;
            default: state_copy_table<0>(p, t); break;
        }
    }
}

__global__ void state_cursor_kernel(const uint32_t* __restrict__ keys, int64_t n, int32_t n_nodes, int32_t K,
                                    int32_t* __restrict__ pos) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = keys[j];
        if (v >= (uint32_t)n_nodes || (j + 1 < n && keys[j + 1] == v)) continue;  // run tails only
        const int64_t m = j + 1 - first_geq(keys, n, v);
        pos[v] = (int32_t)(((int64_t)pos[v] + m) % K);
    }
}

struct StatePlan {
    int bits = 0, passes = 1;
    uint64_t ntiles = 0;
    uint32_t* kbuf[2] = {nullptr, nullptr};
    uint32_t* vbuf[2] = {nullptr, nullptr};
    uint32_t* keys0 = nullptr;
    uint32_t* counts = nullptr;
    uint64_t* partial = nullptr;
    int64_t* dst = nullptr;
    size_t bytes = 0;
};

static StatePlan plan_state(int64_t n, int32_t n_nodes, void* ws) {
    StatePlan p;
    // keys take values 0..n_nodes (sentinel included)
    p.bits = 32 - __builtin_clz((unsigned)n_nodes | 1u);
    p.passes = std::max(1, (p.bits + 7) / 8);
    p.ntiles = ((uint64_t)n + kRadixTile - 1) / kRadixTile;
    const size_t m = (size_t)std::max<int64_t>(n, 1);
    Carve c(ws);
    p.keys0 = c.take<uint32_t>(m);
    for (int b = 0; b < 2; ++b) {
        p.kbuf[b] = c.take<uint32_t>(m);
        p.vbuf[b] = c.take<uint32_t>(m);
    }
    p.counts = c.take<uint32_t>((size_t)kRadixBins * std::max<uint64_t>(p.ntiles, 1));
    p.partial = c.take<uint64_t>(scan_workspace_bytes((int64_t)(kRadixBins * std::max<uint64_t>(p.ntiles, 1))) /
                                 sizeof(uint64_t));
    p.dst = c.take<int64_t>(m);
    p.bytes = c.bytes();
    return p;
}

int read_and_clear_state_err(cudaStream_t st, int* bits) {
    int* dptr = nullptr;
    if (cudaGetSymbolAddress((void**)&dptr, g_state_err) != cudaSuccess) return TGL_ECUDA;
    if (cudaMemcpyAsync(bits, dptr, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess) return TGL_ECUDA;
    if (cudaMemsetAsync(dptr, 0, sizeof(int), st) != cudaSuccess) return TGL_ECUDA;
    return TGL_OK;
}

}  // namespace tgl

using namespace tgl;

extern "C" int tgl_state_write_workspace(int64_t n_events, int32_t n_nodes, size_t* bytes) {
    if (!bytes || n_events < 0 || n_nodes < 0 || n_events >= (int64_t(1) << 31)) return TGL_EINVAL;
    *bytes = plan_state(n_events, n_nodes, nullptr).bytes;
    return TGL_OK;
}

extern "C" int tgl_state_write(const int32_t* ids, const float* ts, int64_t n_events, int32_t n_nodes, int32_t K,
                               int32_t* pos, float* ts_table, const tgl_state_table* tables, int32_t n_tables,
                               void* workspace, size_t ws_bytes, void* stream) {
    NvtxRange nvtx_("tgl_state_write");
    if (n_events < 0 || n_nodes < 0 || n_events >= (int64_t(1) << 31) || K < 1) return TGL_EINVAL;
    if (n_tables < 0 || n_tables > TGL_MAX_GATHER_TABLES || (n_tables > 0 && !tables)) return TGL_EINVAL;
    if (K > 1 && !pos) return TGL_EINVAL;
    if (n_events > 0 && (!ids || !workspace || (ts_table && !ts))) return TGL_EINVAL;
    if ((int64_t)n_nodes * K >= (int64_t(1) << 40)) return TGL_EINVAL;
    StateParams sp;
    memset(&sp, 0, sizeof(sp));
    for (int j = 0; j < n_tables; ++j) {
        const tgl_state_table& t = tables[j];
        if (t.row_bytes <= 0 || (n_events > 0 && (!t.rows || !t.table))) return TGL_EINVAL;
        const uint32_t vs = vec_shift_for(t.row_bytes, t.rows, t.table);
        sp.t[j].rows = static_cast<const unsigned char*>(t.rows);
        sp.t[j].table = static_cast<unsigned char*>(t.table);
        sp.t[j].vec_shift = vs;
        sp.t[j].chunks_per_row = (uint32_t)(t.row_bytes >> vs);
    }
    int rc = check_device();
    if (rc) return rc;
    if (n_events == 0) return TGL_OK;
    StatePlan p = plan_state(n_events, n_nodes, workspace);
    if (ws_bytes < p.bytes) return TGL_EWORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned blocks = (unsigned)std::min<int64_t>((n_events + 255) / 256, 148 * 8);
    state_keys_kernel<<<blocks, 256, 0, st>>>(ids, n_events, n_nodes, p.keys0);
    // S2: stable LSD passes, (key, event index); pass 0 reads keys0 with identity values
    Stream s{nullptr, nullptr, nullptr, nullptr, 0};
    const unsigned grid = (unsigned)p.ntiles;
    for (int pass = 0; pass < p.passes; ++pass) {
        const int shift = 8 * pass;
        const int nb = std::min(8, std::max(0, p.bits - shift));
        const uint32_t mask = (1u << nb) - 1u;
        const uint32_t* kin = pass == 0 ? p.keys0 : p.kbuf[(pass - 1) & 1];
        const uint32_t* vin = pass == 0 ? nullptr : p.vbuf[(pass - 1) & 1];
        if (pass == 0)
            radix_upsweep_kernel<kSrcKeys><<<grid, kRadixThreads, 0, st>>>(s, kin, (uint64_t)n_events, shift, mask,
                                                                             p.counts, p.ntiles);
        else
            radix_upsweep_kernel<kSrcKV><<<grid, kRadixThreads, 0, st>>>(s, kin, (uint64_t)n_events, shift, mask,
                                                                           p.counts, p.ntiles);
        if (cuda_rc(exclusive_scan<uint32_t, uint32_t>(p.counts, p.counts, (int64_t)kRadixBins * p.ntiles,
                                                       (uint32_t*)nullptr, p.partial, st)))
            return TGL_ECUDA;
        if (pass == 0)
            radix_downsweep_kernel<kSrcKeys, kDstKV><<<grid, kRadixThreads, 0, st>>>(
                s, kin, vin, (uint64_t)n_events, shift, mask, p.counts, p.ntiles, p.kbuf[pass & 1], p.vbuf[pass & 1],
                nullptr, nullptr, nullptr, nullptr);
        else
            radix_downsweep_kernel<kSrcKV, kDstKV><<<grid, kRadixThreads, 0, st>>>(
                s, kin, vin, (uint64_t)n_events, shift, mask, p.counts, p.ntiles, p.kbuf[pass & 1], p.vbuf[pass & 1],
                nullptr, nullptr, nullptr, nullptr);
    }
    const uint32_t* keys = p.kbuf[(p.passes - 1) & 1];
    const uint32_t* evt = p.vbuf[(p.passes - 1) & 1];
    state_slot_kernel<<<blocks, 256, 0, st>>>(keys, evt, n_events, n_nodes, K, pos, ts, ts_table, p.dst);
    if (n_tables > 0) {
        sp.keys = keys;
        sp.evt = evt;
        sp.dst = p.dst;
        sp.n = n_events;
        sp.n_tables = n_tables;
        uint64_t work = 0;
        for (int j = 0; j < n_tables; ++j) work = std::max<uint64_t>(work, (uint64_t)n_events * sp.t[j].chunks_per_row);
        const uint64_t g = std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, 148ull * 8));
        state_copy_kernel<<<(unsigned)g, 256, 0, st>>>(sp);
    }
    if (K > 1) state_cursor_kernel<<<blocks, 256, 0, st>>>(keys, n_events, n_nodes, K, pos);
    return cudaGetLastError() == cudaSuccess ? TGL_OK : TGL_ECUDA;
}
