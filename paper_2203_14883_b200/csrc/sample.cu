// sample.cu -- the parallel temporal sampler of TGL (Alg. 1) on B200.
//
// Per layer chain (layer 0: one chain covering all S dynamic snapshots of a root, whose S+1 cuts
// share the indptr pair and narrow each other's range; layer l >= 1: one chain per snapshot s whose
// roots are block (l-1, s)'s outputs, Alg. 1, R#3) three kernels run on the caller's
// stream, with no inter-CTA waiting anywhere (measured faster on B200 than one fused kernel with a
// decoupled look-back, whose tiles wait on slow predecessors: profiles/r01):
//
//   K4a window_kernel  one lane per root: node record (bounds + 14 fence timestamps, read by 4
//                      cooperating lanes), S+1 cut searches (lower_bound) inside their fence gaps
//                      of the node's time-sorted ts list -- the stateless replacement of the
//                      paper's per-node pointers pt_0..pt_S (Sec. 3.1 "Sampling", L260-L262) --
//                      through the 16-ary index (tsindex.cuh) for long gaps.  Writes per root the
//                      S+1 cuts and per (snapshot, 256-root tile) the edge count min(k, c):
//                      most_recent -> the min(k, c) "closest to the end pointer";
//                      uniform -> a uniform min(k, c)-subset (R#5).
//   (K5) tile bases   the window kernel also adds its tile totals into per-64-tile super totals
//                      and per-4096-tile hyper totals (integer atomics: order-independent, so
//                      deterministic); a copy CTA sums the hyper, super and tile totals before it
//                      (<= 3 x 63 + hyper loads) -- no scan kernel, no waiting.
//   K4b copy_kernel    one warp per 32 roots: warp scan of its counts + tile base -> offsets[i];
//                      uniform: Floyd's k-subset with Philox4x32-10 draws, ascending (R#5, R#6);
//                      then the tile's outputs are copied as one flat range per snapshot -- lane o
//                      finds its root by a 5-step search over the warp's inclusive counts -- loading
//                      the selected slot record {ts, nbr, eid} (16 bytes, or 8 packed: one load per output, one request per run of
//                      slots) and storing (nbr, eid, dt[, ts_edge, child key, child lo]) as
//                      coalesced runs (a9, a10; K6 fused).
// dt = t_root (-) t_edge with __fsub_rn; window bounds with __fmul_rn / __fsub_rn (R#12).
// Everything strictly before the root: ts < U = t.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "chain.cuh"
#include "common.cuh"
#include "scan.cuh"
#include "tsindex.cuh"

namespace tgl {

#ifndef TGL_WINDOW_MINB
#define TGL_WINDOW_MINB 8
#endif
#ifndef TGL_COPY_MINB
#define TGL_COPY_MINB 6  // uniform copy (Floyd picks): 40 registers
#endif
#ifndef TGL_COPY_MINB_MR
#define TGL_COPY_MINB_MR 8  // most_recent copy: 32 registers, no spills (C5 +6 %)
#endif
constexpr int kTile = 256;  // roots per tile (one lane per root)
constexpr int kWarps = kTile / 32;
#ifndef TGL_COPY_UNROLL
#define TGL_COPY_UNROLL 2  // most_recent (C5: 1 / 3 / 4 slower, profiles/r02/experiments/codec_copy_unroll_C5.txt)
#endif
#ifndef TGL_COPY_UNROLL_UNI
#define TGL_COPY_UNROLL_UNI 2
#endif
constexpr int kSuperShift = 6;  // 64 tiles per super tile (tile bases: super totals + tile totals)
#ifndef TGL_INDEX_MIN
#define TGL_INDEX_MIN 128  // r02 C4 window: 128 388 us, 512 401, 4096 407 (C5 unchanged); r01 kernels preferred 4096
#endif
constexpr uint32_t kIndexMin = TGL_INDEX_MIN;  // gaps longer than this descend the 16-ary index
constexpr int kPicksSmemPerWarp = 8 * 1024;  // bytes of uniform picks kept in shared memory per warp

struct BlockOut {
    int64_t* offsets;
    int32_t* nbr;
    int32_t* eid;
    float* dt;
    float* ts_edge;       // may be null
    uint64_t* child_key;  // may be null
    float* child_lo;      // may be null
    float* child_t;       // hop roots' times under TGL_HOP_ROOT_TIME (R#23), else null
    int64_t* n_roots_dev;
    int64_t* nnz_dev;
};

// Fused gather (Fig. 2 step 2): the copy kernel also copies, for every output
// it writes, the row of its source node (node memory / mailbox / their times) or of its edge (edge
// features) from caller tables into caller outputs at the output's index.  Rows that are whole
// 16-byte chunks are copied by the whole warp per output; narrower rows lane per output.
constexpr int kMaxFused = TGL_MAX_FUSED_GATHER;
struct FusedTable {
    const void* table;
    void* out;
    int64_t n_rows;
    uint32_t chunks16;  // row_bytes / 16 when rows are 16-byte chunks (and aligned), else 0
    uint32_t words;     // row_bytes / 4 otherwise
    int32_t by_edge;    // 0: indexed by the output's source node (nbr), 1: by its edge id (eid)
};
struct FusedGather {
    int32_t n;
    FusedTable t[kMaxFused];
};

struct SampleParams {
    const int64_t* indptr;
    const int32_t* nbr;
    const float* ts;
    const int32_t* eid;
    const SlotRec* recs;                    // slot records {ts, nbr, eid, 0} (tsindex.cuh), 8-byte packed, or null
    const int4* nodes;                      // 64-byte node records {lo, hi, 14 fences} (tsindex.cuh), or null
    const float* lvl[kMaxIndexLevels + 1];  // lvl[l] = index level l (1-based)
    int32_t n_levels;                       // 0 -> no index
    // time codec (tsindex.cuh "time codes"): node records hold 54 fence codes and the cut probes
    // read 1-byte codes; packed: 8-byte slot records {nbr | code << bn | eid - eid_base[code]}
    const uint8_t* codes;    // null -> no codec
    const float* tval;       // [256] sorted distinct times (+inf padded)
    const int32_t* tebase;   // [256] eid base per code
    int32_t packed;  // 1: time codes; 2: integer times (tsindex.cuh)
    uint32_t bn, bc;
    int32_t ebase0;  // packed = 2: the smallest eid
    uint32_t n_stored;  // E_s (slot count of the handle's lists)
    int32_t n_nodes;
    int64_t node_lo;  // node-sharded handles: global id of local node 0 (0 otherwise)
    const int32_t* root_node;
    const float* root_ts;
    const uint64_t* root_key;  // explicit root keys (layer 0: caller's, may be null; l >= 1: parent's)
    const float* root_lo;      // l >= 1: inherited lower bounds; null -> -inf
    uint64_t root_key_base;
    int64_t n_roots;                // layer 0: count; l >= 1: capacity
    const int64_t* n_roots_dev_in;  // l >= 1: device count (parent block's nnz)
    int32_t layer, nsb, snap0, k;
    int32_t replacement;  // uniform with replacement (R#24)
    const uint32_t* valid;  // R#28: validity bitmask over edge ids (null: every edge valid)
    uint32_t* vpicks;       // R#28: [nsb][roots_cap][k] selected slots (absolute), ascending
    uint32_t* vtake;        // R#28: [nsb][roots_cap] selected count
    float snapshot_len;
    uint32_t seed_lo, seed_hi;
    uint32_t* cuts;  // [nsb+1][roots_cap] c_0 >= c_1 >= .. >= c_nsb: window b = slots [c_(b+1), c_b)
    uint32_t* tile_tot;    // [nsb][tiles_cap] edges emitted per 256-root tile
    uint64_t* super_tot;   // [nsb][supers_cap] per 64 tiles (integer atomics: order-independent), zeroed per call
    int64_t supers_cap;
    uint64_t* hyper_tot;   // [nsb][hypers_cap] per 64 super tiles (4,096 tiles), same rules
    int64_t hypers_cap;
    int64_t roots_cap, tiles_cap;
    uint32_t* picks_global;  // null -> picks in shared memory; else [tiles_cap * 8 warps][nsb*k][32]
    int* err;
    FusedGather fg;  // optional row gather of the outputs (last layer, one block)
    BlockOut out[TGL_MAX_SNAPSHOTS];
};

__device__ __forceinline__ int64_t chain_roots(const SampleParams& p) {
    int64_t n = p.n_roots;
    if (p.n_roots_dev_in) {
        const int64_t m = *p.n_roots_dev_in;
        n = m < n ? m : n;
    }
    return n > 0 ? n : 0;
}

// Scattered reads of the sampler with an explicit L2 fill size: by default a B200 L2 miss fills
// the whole 128-byte line (4 sectors); the ".L2::64B" qualifier fills 64 bytes (tools/granule.cu:
// 127.7 -> 63.8 DRAM bytes per scattered 4-byte read, same request rate).  Node records are 64
// bytes, cut probes 4 bytes and a root's selected slot records a run of <= k x 12 bytes.
__device__ __forceinline__ float ld_rand_f32(const float* p) {
    float v;
    asm("ld.global.nc.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
// slot records (copy kernel), one aligned load per output: most_recent reads runs of <= k records
// (128-byte fills; 64 / 256: +-1 %, profiles/r02/experiments/recfill_ktime_C5.txt), uniform reads
// scattered single records (64-byte fills: half the DRAM bytes of a line per pick)
template <bool RUNS>
__device__ __forceinline__ int4 ld_rec16(const SlotRec* p) {
    int4 v;
    if (RUNS)
        asm("ld.global.nc.L2::128B.v4.s32 {%0, %1, %2, %3}, [%4];"
            : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else
        asm("ld.global.nc.L2::64B.v4.s32 {%0, %1, %2, %3}, [%4];"
            : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ int4 ld_rand_v4(const int4* p) {
    int4 v;
    asm("ld.global.nc.L2::64B.v4.s32 {%0, %1, %2, %3}, [%4];"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t ld_rand_u8(const uint8_t* p) {
    uint16_t v;
    asm("ld.global.nc.L2::64B.u8 %0, [%1];" : "=h"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ld_rand_v2_64(const uint2* p) {  // scattered single records
    uint2 v;
    asm("ld.global.nc.L2::64B.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ld_rand_v2(const uint2* p) {
    uint2 v;
    asm("ld.global.nc.L2::128B.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

template <typename T>
__device__ __forceinline__ void st_global_u32(T* p, uint32_t v) {
    asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(v));  // outputs are not re-read by the kernel
}

// ---------------------------------------------------------------------------- cut search
// first slot in [a, b) with ts >= x, else b (R#2).  Long lists first descend the 16-ary index
// (tsindex.cuh): per level a binary search over <= 16 consecutive index entries (one 64-byte
// group: one DRAM request + L1 hits); then a binary search over the remaining <= 15 slots.
__device__ __forceinline__ uint32_t lower_bound_ts(const SampleParams& p, uint32_t a, uint32_t b, float x) {
    if (a >= b) return a;
    uint64_t A = a, B = b;
    if (p.n_levels > 0 && B - A > kIndexMin) {
        int l = 1;
        while (l < p.n_levels && ((B + (1ull << (kIndexShift * l)) - 1) >> (kIndexShift * l)) -
                                         ((A + (1ull << (kIndexShift * l)) - 1) >> (kIndexShift * l)) >
                                     16)
            ++l;
        for (; l >= 1; --l) {
            const int sh = kIndexShift * l;
            const uint64_t j0 = (A + (1ull << sh) - 1) >> sh, j1 = (B + (1ull << sh) - 1) >> sh;
            if (j1 <= j0) continue;
            const float* L = p.lvl[l];
            uint64_t lo = j0, hi = j1;  // first index entry >= x
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if (__ldg(L + mid) < x)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            const uint64_t m = lo - j0;  // entries < x
            if (m > 0) A = ((j0 + m - 1) << sh) + 1;
            if (j0 + m < j1) B = (j0 + m) << sh;
        }
    }
    uint32_t lo = (uint32_t)A, hi = (uint32_t)B;
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        TGL_CHECK(mid < p.n_stored);
        if (ld_rand_f32(p.ts + mid) < x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Up to 4 cuts searched together, cut j in [a[j], b[j]] (a fence gap, or the whole list); called
// by all 32 lanes of the warp (lanes with nothing to search pass empty gaps):
// interleaved binary searches, one independent probe per live cut per step, so a root costs
// max(log2 gap) dependent steps instead of the sum over cuts.  Gaps longer than kIndexMin (hub
// lists) descend the 16-ary index first.
__device__ __forceinline__ void lower_bound_multi(const SampleParams& p, uint32_t (&a)[4], uint32_t (&b)[4],
                                                  const float (&x)[4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (p.n_levels > 0 && b[j] - a[j] > kIndexMin) b[j] = a[j] = lower_bound_ts(p, a[j], b[j], x[j]);
    // a gap of g slots needs ceil(log2(g + 1)) halvings: the warp runs its lanes' maximum as a
    // counted loop (no per-step liveness vote), every cut stepping branch-free while a < b
    uint32_t g = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) g = max(g, b[j] - a[j]);
    const int steps = 32 - __clz((int)__reduce_max_sync(kFull, g));  // all 32 lanes call this
    for (int it = 0; it < steps; ++it) {
        float v[4];
        uint32_t mid[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            mid[j] = a[j] + ((b[j] - a[j]) >> 1);
            TGL_CHECK(a[j] >= b[j] || mid[j] < p.n_stored);
            v[j] = a[j] < b[j] ? ld_rand_f32(p.ts + mid[j]) : 0.0f;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool go = a[j] < b[j], lt = v[j] < x[j];
            a[j] = go && lt ? mid[j] + 1 : a[j];
            b[j] = go && !lt ? mid[j] : b[j];
        }
    }
}

// The same searches over the time codes: cut j = first slot in [a[j], b[j]] whose code is >= q[j]
// (q[j] = #{dictionary times < x[j]}, so code < q[j] <=> ts < x[j]); 64 slots per 64-byte atom.
__device__ __forceinline__ void lower_bound_multi_codes(const SampleParams& p, uint32_t (&a)[4], uint32_t (&b)[4],
                                                        const float (&x)[4], uint32_t q4) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (p.n_levels > 0 && b[j] - a[j] > kIndexMin) b[j] = a[j] = lower_bound_ts(p, a[j], b[j], x[j]);
    uint32_t g = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) g = max(g, b[j] - a[j]);
    const int steps = 32 - __clz((int)__reduce_max_sync(kFull, g));  // all 32 lanes call this
    for (int it = 0; it < steps; ++it) {
        uint32_t v[4], mid[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            mid[j] = a[j] + ((b[j] - a[j]) >> 1);
            TGL_CHECK(a[j] >= b[j] || mid[j] < p.n_stored);
            v[j] = a[j] < b[j] ? ld_rand_u8(p.codes + mid[j]) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool go = a[j] < b[j], lt = v[j] < ((q4 >> (8 * j)) & 0xffu);
            a[j] = go && lt ? mid[j] + 1 : a[j];
            b[j] = go && !lt ? mid[j] : b[j];
        }
    }
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// ---------------------------------------------------------------------------- R#28 validity
// With an edge-validity bitmask ("invalid edges could be simply ignored") the
// candidates of window [a, e) are its slots whose edge is valid.  The window kernel then selects
// explicitly: most_recent walks back from the end pointer collecting the last k valid slots;
// uniform counts the valid slots, draws ranks (Floyd / with replacement, the same Philox counters)
// and maps them to slots in one forward walk.  The copy kernel reads the selected slots.
// uniform draws (R#6): draw j is word j mod 4 of Philox4x32-10 at counter (j / 4, l << 16 | s, rk)
__device__ __forceinline__ uint32_t draw_word(const uint4& r, uint32_t j) {
    const uint32_t q = j & 3u;
    return q == 0 ? r.x : q == 1 ? r.y : q == 2 ? r.z : r.w;
}

template <int STRATEGY>
__device__ __forceinline__ uint32_t select_valid(const SampleParams& p, int64_t i, int b, uint32_t a, uint32_t e,
                                                uint64_t rk) {
    const uint32_t k = (uint32_t)p.k;
    uint32_t* pk = p.vpicks + ((size_t)b * p.roots_cap + i) * k;
    auto ok = [&](uint32_t s) {
        const uint32_t id = (uint32_t)__ldg(p.eid + s);
        return (__ldg(p.valid + (id >> 5)) >> (id & 31)) & 1u;
    };
    uint32_t take = 0;
    if (STRATEGY == TGL_MOST_RECENT) {
        for (uint32_t s = e; s > a && take < k; --s)
            if (ok(s - 1)) pk[k - 1 - take++] = s - 1;  // filled from the back: ascending
        for (uint32_t q = 0; q < take; ++q) pk[q] = pk[k - take + q];
    } else {
        uint32_t cv = 0;
        for (uint32_t s = a; s < e; ++s) cv += ok(s);
        const uint32_t ctr1 = ((uint32_t)p.layer << 16) | (uint32_t)(p.layer == 0 ? b : p.snap0);
        uint4 rnd = make_uint4(0u, 0u, 0u, 0u);
        if (p.replacement) {
            take = cv ? k : 0u;
            for (uint32_t j = 0; j < take; ++j) {
                if ((j & 3u) == 0)
                    rnd = philox4x32_10(make_uint4(j >> 2, ctr1, (uint32_t)rk, (uint32_t)(rk >> 32)), p.seed_lo, p.seed_hi);
                pk[j] = __umulhi(draw_word(rnd, j), cv);
            }
        } else if (cv <= k) {
            take = cv;
            for (uint32_t q = 0; q < cv; ++q) pk[q] = q;
        } else {
            take = k;
            for (uint32_t j = 0; j < k; ++j) {  // Floyd over the ranks (R#5, R#6)
                const uint32_t m = cv - k + j;
                if ((j & 3u) == 0)
                    rnd = philox4x32_10(make_uint4(j >> 2, ctr1, (uint32_t)rk, (uint32_t)(rk >> 32)), p.seed_lo, p.seed_hi);
                const uint32_t r = __umulhi(draw_word(rnd, j), m + 1u);
                bool taken = false;
                for (uint32_t q = 0; q < j; ++q) taken |= pk[q] == r;
                pk[j] = taken ? m : r;
            }
        }
        for (uint32_t j = 1; j < take; ++j) {  // ascending ranks (R#13)
            const uint32_t xj = pk[j];
            int q = (int)j - 1;
            while (q >= 0 && pk[q] > xj) {
                pk[q + 1] = pk[q];
                --q;
            }
            pk[q + 1] = xj;
        }
        uint32_t r = 0, cnt = 0;  // ranks -> slots
        for (uint32_t s = a; s < e && r < take; ++s) {
            if (!ok(s)) continue;
            while (r < take && pk[r] == cnt) pk[r++] = s;
            ++cnt;
        }
    }
    p.vtake[(size_t)b * p.roots_cap + i] = take;
    return take;
}

// word w of a node record parked in shared memory with its 16-byte chunks swizzled by sw
__device__ __forceinline__ float rec_word(const float* rec, int sw, int w) {
    return rec[(((w >> 2) ^ sw) << 2) | (w & 3)];
}

// ---------------------------------------------------------------------------- K4a windows
// TC: the graph has the time codec (node records with 54 fence codes, cut probes over codes)
template <int STRATEGY, bool VALID, bool TC>
__global__ void __launch_bounds__(kTile, VALID ? 6 : TGL_WINDOW_MINB) window_kernel(const __grid_constant__ SampleParams p) {
    __shared__ uint32_t s_red[TGL_MAX_SNAPSHOTS][kWarps];
    __shared__ int4 s_rec[kTile * 4];  // the tile's 64-byte node records (16 KB)
    __shared__ float s_tval[TC ? 256 : 1];  // the codec's sorted distinct times (+inf padded)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n = chain_roots(p);
    const int64_t tile = (int64_t)blockIdx.x;
    const int64_t base_i = tile * kTile;
    if (base_i >= n) return;  // capacity-sized grid (l >= 1): tiles past the end do nothing
    const int64_t i = base_i + threadIdx.x;
    const bool valid = i < n;
    const int nsb = p.nsb;
    const uint32_t k = (uint32_t)p.k;

    // the root loads are issued before the codec dictionary's barrier, so the two overlap
    int32_t rn = 0;
    float t = 0.0f, lin_raw = -INFINITY;
    if (valid) {
        rn = p.root_node[i];
        t = p.root_ts[i];
        if (p.layer > 0 && p.root_lo) lin_raw = p.root_lo[i];
    }
    if (TC) {
        s_tval[threadIdx.x] = __ldg(p.tval + threadIdx.x);  // kTile == 256 entries
        __syncthreads();
    }
    int32_t v = 0;
    bool ok = false;
    if (valid) {
        const int64_t vg = (int64_t)rn - p.node_lo;  // shard-local node id
        v = (int32_t)vg;
        if (vg < 0 || vg >= (int64_t)p.n_nodes)
            atomicOr(p.err, kErrRange);
        else if (!isfinite(t))
            atomicOr(p.err, kErrInval);
        else
            ok = true;
    }
    const float lin = ok ? lin_raw : -INFINITY;
    // the root key (R#7), needed here only by the validity path's uniform draws
    const uint64_t rk0 = (VALID && STRATEGY == TGL_UNIFORM && valid)
                             ? (p.root_key ? p.root_key[i] : p.root_key_base + (uint64_t)i) : 0ull;
    // the cut times searched through the fences: all S+1 cuts of a layer-0 root with finite t_s and
    // S <= 3 (c_0 = t, c_j = t (-) (j (x) t_s)); otherwise U = t and the first window's lower bound
    const bool multi = nsb <= 3 && p.layer == 0 && isfinite(p.snapshot_len);
    auto cuts_of = [&](float tr, float lr, float (&x)[4]) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (multi)
                x[j] = j == 0 ? tr : (j <= nsb ? __fsub_rn(tr, __fmul_rn((float)j, p.snapshot_len)) : -INFINITY);
            else
                x[j] = j == 0 ? tr : (j == 1 ? (p.layer == 0 ? __fsub_rn(tr, p.snapshot_len) : lr) : -INFINITY);
        }
    };
    float x[4];
    cuts_of(t, lin, x);
    uint32_t lo = 0, hi = 0, ga[4], gb[4];  // cut j lies in [ga[j], gb[j]]
    uint32_t xq = 0;                        // TC: code thresholds of x[j] (byte j)
    bool early;                             // some slot is earlier than t: the list must be searched
    if (p.nodes) {
        // 4 lanes read one 64-byte node record (one request per record): rounds q = 0..3 cover the
        // warp's roots q*8 .. q*8+7 and park the records in shared memory (16-byte chunk c of root r
        // at chunk slot c ^ ((r >> 1) & 3): the 8 lanes of a quarter-warp then read 8 distinct
        // bank groups); then every lane counts its own root's 14 fences below each cut time with a
        // branch-free binary search over the record (fences are sorted)
        int4* wrec = s_rec + warp * 32 * 4;
        const int quad = lane >> 2, part = lane & 3;
        int4 ch[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int src = q * 8 + quad;
            const int vq = __shfl_sync(kFull, v, src);
            const bool okq = __shfl_sync(kFull, ok, src);
            // an invalid root reads as an empty list: lo = hi = 0, every fence +inf
            constexpr int kInfW = TC ? 0x7f7f7f7f : 0x7f800000;
            ch[q] = okq ? ld_rand_v4(p.nodes + (size_t)vq * 4 + part)
                        : make_int4(part ? kInfW : 0, part ? kInfW : 0, kInfW, kInfW);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int src = q * 8 + quad;
            wrec[src * 4 + (part ^ ((src >> 1) & 3))] = ch[q];
        }
        __syncwarp();
        const int sw = (lane >> 1) & 3;
        const float* rec = reinterpret_cast<const float*>(wrec + lane * 4);
        lo = __float_as_uint(rec_word(rec, sw, 0));
        hi = __float_as_uint(rec_word(rec, sw, 1));
        const uint32_t d = hi - lo;
        uint32_t packed = 0;
        if (TC) {
            // code thresholds q[j] = #{dictionary times < x[j]} (7 halvings over 128 padded
            // entries).  Chronological roots give a warp one root time (and one inherited bound)
            // in the usual case: then lanes 0..3 search one cut each and broadcast.
            const float t0 = __shfl_sync(kFull, t, 0), l0 = __shfl_sync(kFull, lin, 0);
            if (__all_sync(kFull, t == t0 && lin == l0)) {
                const int jj = lane & 3;
                const float xs = jj == 0 ? x[0] : jj == 1 ? x[1] : jj == 2 ? x[2] : x[3];
                uint32_t qc = 0;
#pragma unroll
                for (int step = 64; step >= 1; step >>= 1) qc += s_tval[qc + step - 1] < xs ? step : 0u;
#pragma unroll
                for (int j = 0; j < 4; ++j) xq |= __shfl_sync(kFull, qc, j) << (8 * j);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t qc = 0;
#pragma unroll
                    for (int step = 64; step >= 1; step >>= 1) qc += s_tval[qc + step - 1] < x[j] ? step : 0u;
                    xq |= qc << (8 * j);
                }
            }
            // #fences < q = 5 c1 + c2 (tsindex.cuh): SWAR byte compares of 7-bit codes -- byte b of
            // (((q-1) x 0x01) | 0x80) - w keeps its high bit iff b < q, no borrow crosses bytes
            constexpr uint32_t H = 0x80808080u;
            const uint32_t s0 = __float_as_uint(rec_word(rec, sw, 2)), s1 = __float_as_uint(rec_word(rec, sw, 3)),
                           s2 = __float_as_uint(rec_word(rec, sw, 4));
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t qc = (xq >> (8 * j)) & 0xffu;
                const uint32_t Qm = ((max(qc, 1u) - 1u) * 0x01010101u) | H;  // q = 0: masked below
                const int c1 = __popc((Qm - s0) & H) + __popc((Qm - s1) & H) + __popc((Qm - s2) & H);
                const uint32_t wg = __float_as_uint(rec_word(rec, sw, 5 + c1));
                const int m = qc ? 5 * c1 + __popc((Qm - wg) & H) : 0;
                packed |= (uint32_t)m << (8 * j);
                ga[j] = m ? code_fence_pos(lo, d, m - 1) + 1 : lo;
                gb[j] = m < kCodeFences ? code_fence_pos(lo, d, m) : hi;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                // number of fences f[0..13] (= words 2..15) below x[j]; positions >= 14 act as +inf
                int c = 0;
#pragma unroll
                for (int step = 8; step >= 1; step >>= 1) {
                    const int e = min(c + step - 1, kFences);
                    const float f = rec_word(rec, sw, 2 + min(e, kFences - 1));
                    c += (e < kFences && f < x[j]) ? step : 0;
                }
                packed |= (uint32_t)c << (8 * j);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int m = (int)((packed >> (8 * j)) & 0xffu);
                ga[j] = m ? fence_pos(lo, d, m - 1) + 1 : lo;
                gb[j] = m < kFences ? fence_pos(lo, d, m) : hi;
            }
        }
        early = (packed & 0xffu) != 0;  // f[0] = the first edge time < t
    } else {
        if (ok) {
            lo = (uint32_t)__ldg(p.indptr + v);
            hi = (uint32_t)__ldg(p.indptr + v + 1);
        }
        early = lo < hi && __ldg(p.ts + lo) < t;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            ga[j] = lo;
            gb[j] = x[j] > -INFINITY ? hi : lo;
        }
    }
    if (multi) {
        uint32_t cut[4];
        if (!early) {  // no slot before t: every cut is lo (empty gaps: no probes)
#pragma unroll
            for (int j = 0; j < 4; ++j) ga[j] = gb[j] = lo;
        }
        if (TC && p.nodes)
            lower_bound_multi_codes(p, ga, gb, x, xq);  // the whole warp: its step count is a warp reduction
        else
            lower_bound_multi(p, ga, gb, x);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            cut[j] = ga[j];
            TGL_CHECK(!valid || (lo <= cut[j] && cut[j] <= hi && hi <= p.n_stored));
        }
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            if (b >= nsb) break;
            const uint32_t c = cut[b] - cut[b + 1];
            const uint32_t take = VALID ? (valid ? select_valid<STRATEGY>(p, i, b, cut[b + 1], cut[b], rk0) : 0u)
                                          : (p.replacement ? (c ? k : 0u) : (c < k ? c : k));
            if (valid) {
                if (b == 0) p.cuts[i] = cut[0];
                p.cuts[(size_t)(b + 1) * p.roots_cap + i] = cut[b + 1];
            }
            const uint32_t s2 = __reduce_add_sync(kFull, take);
            if (lane == 0) s_red[b][warp] = s2;
        }
    } else {
        uint32_t bcur = early ? lower_bound_ts(p, ga[0], gb[0], t) : lo;
        for (int b = 0; b < nsb; ++b) {
            // lower bound of window b: layer 0 -> t (-) ((b+1) (x) t_s); l >= 1 -> inherited
            const float xb = p.layer == 0 ? __fsub_rn(t, __fmul_rn((float)(b + 1), p.snapshot_len)) : lin;
            uint32_t a = lo;
            if (xb > -INFINITY && bcur > lo) {  // empty window when the element before the cut is < x
                if (b == 0)                      // the first lower bound's fence gap (x[1] = xb)
                    a = min(lower_bound_ts(p, min(ga[1], bcur), min(gb[1], bcur), xb), bcur);
                else
                    a = ld_rand_f32(p.ts + bcur - 1) < xb ? bcur : lower_bound_ts(p, lo, bcur - 1, xb);
            }
            const uint32_t c = bcur - a;
            const uint32_t take = VALID ? (valid ? select_valid<STRATEGY>(p, i, b, a, bcur, rk0) : 0u)
                                          : (p.replacement ? (c ? k : 0u) : (c < k ? c : k));
            if (valid) {
                if (b == 0) p.cuts[i] = bcur;
                p.cuts[(size_t)(b + 1) * p.roots_cap + i] = a;
            }
            const uint32_t s2 = __reduce_add_sync(kFull, take);
            if (lane == 0) s_red[b][warp] = s2;
            bcur = a;
        }
    }
    __syncthreads();
    if (threadIdx.x < nsb) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += s_red[threadIdx.x][w];
        p.tile_tot[(size_t)threadIdx.x * p.tiles_cap + tile] = s;
        // super / hyper totals are read only for super tiles BEFORE a copy CTA's own: a grid of one
        // super tile (per-batch calls) neither zeroes nor accumulates them
        if (gridDim.x > (1u << kSuperShift)) {
            atomicAdd(reinterpret_cast<unsigned long long*>(p.super_tot + (size_t)threadIdx.x * p.supers_cap +
                                                            (tile >> kSuperShift)),
                      (unsigned long long)s);
            atomicAdd(reinterpret_cast<unsigned long long*>(p.hyper_tot + (size_t)threadIdx.x * p.hypers_cap +
                                                            (tile >> (2 * kSuperShift))),
                      (unsigned long long)s);
        }
    }
    // programmatic dependent launch: the copy kernel may be scheduled once every window CTA got
    // here (its griddepcontrol.wait still waits for this grid's completion and memory flush)
    asm volatile("griddepcontrol.launch_dependents;");
}

// Floyd's k-subset for k <= kFloydRegs with the picks in registers (R#5, R#6): draw j is word j
// mod 4 of Philox4x32-10 at counter (j / 4, ctr1, rk); r_j = floor(x_j (m_j + 1) / 2^32),
// m_j = c - k + j; pick j = r_j unless an earlier pick equals it, else m_j (> every earlier pick).
// The picks are kept ascending (R#13) by a compare-exchange chain after each draw (static register
// indices) and stored at pk[0..k) (the window's place in the warp's flat output order).  Same set
// and order as the shared-memory insertion below -- which ran each draw's shift loop at the warp's
// slowest lane.
constexpr int kFloydRegs = 16;
__device__ __forceinline__ void floyd_in_registers(uint32_t* pk, uint32_t len, int k, uint32_t ctr1, uint64_t rk,
                                                   uint32_t seed_lo, uint32_t seed_hi) {
    uint32_t a[kFloydRegs];
    uint4 rnd = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int j = 0; j < kFloydRegs; ++j) {
        a[j] = 0xffffffffu;
        if (j < k) {
            if ((j & 3) == 0)
                rnd = philox4x32_10(make_uint4((uint32_t)j >> 2, ctr1, (uint32_t)rk, (uint32_t)(rk >> 32)), seed_lo,
                                    seed_hi);
            const uint32_t m = len - (uint32_t)k + (uint32_t)j;
            const uint32_t r = __umulhi(draw_word(rnd, (uint32_t)j), m + 1u);
            bool taken = false;
#pragma unroll
            for (int i = 0; i < j; ++i) taken |= a[i] == r;
            a[j] = taken ? m : r;
            // keep a[0..j] ascending: one compare-exchange chain bubbles the new pick into place
#pragma unroll
            for (int i = j - 1; i >= 0; --i) {
                const uint32_t lo = min(a[i], a[i + 1]), hi = max(a[i], a[i + 1]);
                a[i] = lo;
                a[i + 1] = hi;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < kFloydRegs; ++j)
        if (j < k) pk[j] = a[j];
}

// the fused gather of one group of (up to 32) outputs held one per lane
__device__ __forceinline__ void fused_gather_rows(const SampleParams& p, bool act, int64_t gi, int32_t nbr,
                                                  int32_t eid, int lane) {
    for (int j = 0; j < p.fg.n; ++j) {
        const FusedTable& T = p.fg.t[j];
        const int32_t id = T.by_edge ? eid : nbr;
        const bool inr = id >= 0 && (int64_t)id < T.n_rows;
        if (act && !inr && id != -1) atomicOr(p.err, kErrRange);  // as tgl_gather: zero row + ERANGE
        if (T.chunks16) {  // whole warp per output row, 16-byte chunks
            uint32_t m = __ballot_sync(kFull, act);
            while (m) {
                const int q = __ffs(m) - 1;
                m &= m - 1;
                const int32_t idq = __shfl_sync(kFull, id, q);
                const int64_t gq = __shfl_sync(kFull, gi, q);
                const bool okq = __shfl_sync(kFull, inr, q);
                const int4* src = reinterpret_cast<const int4*>(T.table) + (int64_t)idq * T.chunks16;
                int4* dst = reinterpret_cast<int4*>(T.out) + gq * T.chunks16;
                for (uint32_t c = lane; c < T.chunks16; c += 32) dst[c] = okq ? __ldg(src + c) : make_int4(0, 0, 0, 0);
            }
        } else if (act) {  // narrow rows (e.g. one timestamp): lane per output
            const int32_t* src = reinterpret_cast<const int32_t*>(T.table) + (int64_t)id * T.words;
            int32_t* dst = reinterpret_cast<int32_t*>(T.out) + gi * T.words;
            for (uint32_t w = 0; w < T.words; ++w) dst[w] = inr ? __ldg(src + w) : 0;
        }
    }
}

// ---------------------------------------------------------------------------- K4b copy
// Per warp shared memory (words): inclusive counts [nsb][32]; segment list [nsb*32] of uint2
// {start << 9 | b << 5 | r, first slot} (the warp's non-empty (block, root) windows in output
// order); root times [32]; root keys [32] (u64); per-block output pointers pre-offset to the
// warp's first output {nbr, eid, dt, pad} (u64 each); uniform picks [nsb][k][32].
__host__ __device__ inline int copy_warp_words(int nsb, int k, bool picks_in_smem) {
    return nsb * 32 + 2 * nsb * 32 + 32 + 2 * 32 + 8 * nsb + (picks_in_smem ? nsb * k * 32 : 0);
}

// PSMEM: uniform picks in shared memory (known at compile time, so LDS/STS instead of generic
// 64-bit accesses); else in the global workspace
// PK: 8-byte packed slot records of the time codec (decoded through the dictionaries, which sit
// behind the warps' areas in dynamic shared memory: 2 KB)
template <int STRATEGY, bool VALID, int OUTX, bool PSMEM, int PK>
__global__ void __launch_bounds__(kTile, OUTX == 2 ? 6 : (STRATEGY == TGL_MOST_RECENT ? TGL_COPY_MINB_MR : TGL_COPY_MINB)) copy_kernel(const __grid_constant__ SampleParams p) {
    constexpr bool EXTRA = OUTX == 1;   // per-output data for a following layer / dedup
    constexpr bool GATHER = OUTX == 2;  // fused row gather of the last layer's outputs
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ uint32_t s_wsum[TGL_MAX_SNAPSHOTS][kWarps];
    __shared__ uint64_t s_tbase[TGL_MAX_SNAPSHOTS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n = chain_roots(p);
    const int64_t tile = (int64_t)blockIdx.x;
    const int64_t base_i = tile * kTile;
    if (n == 0) {  // empty chain: the first CTA writes the empty blocks
        if (tile == 0 && threadIdx.x < p.nsb) {
            p.out[threadIdx.x].offsets[0] = 0;
            *p.out[threadIdx.x].nnz_dev = 0;
            *p.out[threadIdx.x].n_roots_dev = 0;
        }
        return;
    }
    if (base_i >= n) return;
    const int64_t i = base_i + threadIdx.x;
    const bool valid = i < n;
    const int nsb = p.nsb;
    const int k = p.k;
    constexpr bool picks_smem = STRATEGY == TGL_UNIFORM && PSMEM;
    uint32_t* ws = smem + warp * copy_warp_words(nsb, k, picks_smem);
    uint32_t* inc = ws;                                                   // [nsb][32]
    uint2* seg = reinterpret_cast<uint2*>(inc + nsb * 32);                // [nsb * 32]
    float* troot = reinterpret_cast<float*>(seg + nsb * 32);              // [32]
    uint64_t* rkey = reinterpret_cast<uint64_t*>(troot + 32);             // [32] (even word offset)
    uint64_t* wptr = rkey + 32;                                           // [nsb][4]
    uint32_t* picks = nullptr;
    if (STRATEGY == TGL_UNIFORM)
        picks = picks_smem ? reinterpret_cast<uint32_t*>(wptr + 4 * nsb)
                           : p.picks_global + ((size_t)tile * kWarps + warp) * nsb * k * 32;

    float* s_tv = reinterpret_cast<float*>(smem + kWarps * copy_warp_words(nsb, k, picks_smem));  // PK only
    int32_t* s_te = reinterpret_cast<int32_t*>(s_tv + 256);
    if (PK == 1) {
        s_tv[threadIdx.x] = __ldg(p.tval + threadIdx.x);  // kTile == 256 entries
        s_te[threadIdx.x] = __ldg(p.tebase + threadIdx.x);
    }
    const float t = valid ? p.root_ts[i] : 0.0f;
    troot[lane] = t;
    uint64_t rk = 0;
    if (STRATEGY == TGL_UNIFORM || EXTRA) {
        rk = p.root_key ? (valid ? p.root_key[i] : 0ull) : p.root_key_base + (uint64_t)i;
        rkey[lane] = rk;
    }
    // everything below reads the window kernel's outputs: wait for that grid (a no-op when the
    // copy kernel was launched without programmatic stream serialisation)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // The prologue's loads -- this root's cuts and, in warps b < nsb, block b's tile-base totals --
    // are issued together: one memory round trip instead of one per cut and per total level.  The
    // copy kernel's CTAs are short (256 roots), so a chain of dependent prologue loads (8 round
    // trips) was half of its time on C5 (208 of 409 us with the flat copy removed).
    constexpr int kPre = 4;  // cuts c_0 .. c_3 prefetched (nsb <= 3: all of them)
    uint32_t cpre[kPre];
#pragma unroll
    for (int j = 0; j < kPre; ++j) cpre[j] = (valid && j <= nsb) ? p.cuts[(size_t)j * p.roots_cap + i] : 0u;
    uint64_t tb_acc = 0;  // warp b < nsb: block b's totals before this tile (lane partial sums)
    {
        const int b = warp;
        if (b < nsb) {
            const int64_t t = tile, sup = t >> kSuperShift, hyp = t >> (2 * kSuperShift);
            // <= 63 super totals and <= 63 tile totals: two lanes' worth each, loaded at once
            const int64_t s0 = (hyp << kSuperShift) + lane, t0 = (sup << kSuperShift) + lane;
            const uint64_t* st = p.super_tot + (size_t)b * p.supers_cap;
            const uint32_t* tt = p.tile_tot + (size_t)b * p.tiles_cap;
            const uint64_t a0 = s0 < sup ? st[s0] : 0ull, a1 = s0 + 32 < sup ? st[s0 + 32] : 0ull;
            const uint32_t a2 = t0 < t ? tt[t0] : 0u, a3 = t0 + 32 < t ? tt[t0 + 32] : 0u;
            for (int64_t q = lane; q < hyp; q += 32) tb_acc += p.hyper_tot[(size_t)b * p.hypers_cap + q];
            tb_acc += a0 + a1 + a2 + a3;
        }
    }
    // counts, warp-local prefix, the segment list; uniform picks
    uint32_t cb = cpre[0];       // c_b
    uint32_t flat = 0, nseg = 0;  // warp outputs / non-empty windows of the blocks before b
    for (int b = 0; b < nsb; ++b) {
        const uint32_t cn = b + 1 < kPre ? (b == 0 ? cpre[1] : b == 1 ? cpre[2] : cpre[3])
                                         : (valid ? p.cuts[(size_t)(b + 1) * p.roots_cap + i] : 0u);  // c_(b+1)
        const uint32_t len = cb - cn;                                                 // window size c
        const uint32_t take = VALID ? (valid ? p.vtake[(size_t)b * p.roots_cap + i] : 0u)
                                    : (p.replacement ? (len ? (uint32_t)k : 0u) : (len < (uint32_t)k ? len : (uint32_t)k));
        // most_recent: the take slots closest to the end pointer; uniform: picks from c_(b+1)
        const uint32_t first = STRATEGY == TGL_MOST_RECENT ? cb - take : cn;
        cb = cn;
        const uint32_t x = warp_incl_scan(take, lane);
        inc[b * 32 + lane] = x;
        const uint32_t wtot = __shfl_sync(kFull, x, 31);
        if (lane == 31) s_wsum[b][warp] = x;
        const uint32_t nz = __ballot_sync(kFull, take > 0);
        const uint32_t fstart = flat + x - take;  // warp-flat index of this window's first output
        if (take > 0)
            seg[nseg + __popc(nz & lanemask_lt())] =
                make_uint2((fstart << 9) | ((uint32_t)b << 5) | (uint32_t)lane, first);
        nseg += __popc(nz);
        flat += wtot;
        if (STRATEGY == TGL_UNIFORM && !VALID) {
            // pick q of this window at picks[fstart + q]: stored in the warp's flat output order, so
            // the copy loop's 32 lanes read 32 consecutive words (the [q][root] layout put a root's
            // picks in one bank: ~10-way conflicts per read, profiles/r02/c4)
            uint32_t* pk = picks + fstart;
            const uint32_t ctr1 = ((uint32_t)p.layer << 16) | (uint32_t)(p.layer == 0 ? b : p.snap0);
            uint4 rnd = make_uint4(0u, 0u, 0u, 0u);
            if (!p.replacement && len <= (uint32_t)k) {
                for (uint32_t q = 0; q < len; ++q) pk[q] = q;
            } else if (p.replacement) {
                // with replacement (R#24): r_j uniform in [0, c) from the counter of Floyd's draw j
                for (uint32_t j = 0; j < take; ++j) {
                    if ((j & 3u) == 0)
                        rnd = philox4x32_10(make_uint4(j >> 2, ctr1, (uint32_t)rk, (uint32_t)(rk >> 32)), p.seed_lo,
                                            p.seed_hi);
                    pk[j] = __umulhi(draw_word(rnd, j), len);
                }
                for (int j = 1; j < (int)take; ++j) {  // ascending slot order (R#13)
                    const uint32_t xj = pk[j];
                    int q = j - 1;
                    while (q >= 0 && pk[q] > xj) {
                        pk[q + 1] = pk[q];
                        --q;
                    }
                    pk[q + 1] = xj;
                }
            } else if (k <= kFloydRegs) {
                // Floyd (R#5, R#6) with the picks in registers: the k draws and their membership
                // tests fully unrolled (k is warp-uniform: no divergence), then a sorting network
                floyd_in_registers(pk, len, k, ctr1, rk, p.seed_lo, p.seed_hi);
            } else {
                // Floyd: for m = c-k .. c-1, r uniform in [0, m]; take r unless taken, else m
                for (int j = 0; j < k; ++j) {
                    const uint32_t m = len - (uint32_t)k + (uint32_t)j;
                    if ((j & 3) == 0)
                        rnd = philox4x32_10(make_uint4((uint32_t)j >> 2, ctr1, (uint32_t)rk, (uint32_t)(rk >> 32)),
                                            p.seed_lo, p.seed_hi);
                    const uint32_t rr = __umulhi(draw_word(rnd, (uint32_t)j), m + 1u);
                    // the picks so far are kept ascending (R#13): one downward pass shifts those
                    // > rr up a slot; if rr is already taken, Floyd takes m instead, which exceeds
                    // every earlier pick (<= m - 1): shift back and append it.  The set -- hence
                    // the output -- is Floyd's; only the sort is merged into the draws.
                    int q = j - 1;
                    uint32_t v = 0;
                    while (q >= 0 && (v = pk[q]) > rr) {
                        pk[q + 1] = v;
                        --q;
                    }
                    if (q >= 0 && v == rr) {
                        for (int u = q + 1; u < j; ++u) pk[u] = pk[u + 1];
                        pk[j] = m;
                    } else {
                        pk[q + 1] = rr;
                    }
                }
            }
        }
    }
    // tile base per snapshot (loaded above): warp b sums the hyper totals before this tile's hyper tile, the super totals
    // before its super tile inside it and the tile totals before it inside its super tile (all
    // final: the window kernel has completed); blocks beyond the warp count (nsb > 8) here
    if (warp < nsb) {
        uint64_t acc = tb_acc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (lane == 0) s_tbase[warp] = acc;
    }
    for (int b = warp + kWarps; b < nsb; b += kWarps) {
        const int64_t t = tile, sup = t >> kSuperShift, hyp = t >> (2 * kSuperShift);
        uint64_t acc = 0;
        for (int64_t q = lane; q < hyp; q += 32) acc += p.hyper_tot[(size_t)b * p.hypers_cap + q];
        for (int64_t q = (hyp << kSuperShift) + lane; q < sup; q += 32) acc += p.super_tot[(size_t)b * p.supers_cap + q];
        for (int64_t q = (sup << kSuperShift) + lane; q < t; q += 32) acc += p.tile_tot[(size_t)b * p.tiles_cap + q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (lane == 0) s_tbase[b] = acc;
    }
    __syncthreads();
    const bool last_tile = base_i + kTile >= n;
    uint32_t fb = 0;  // warp-flat index of block b's first output
    for (int b = 0; b < nsb; ++b) {
        uint64_t wb = s_tbase[b];
        for (int w = 0; w < warp; ++w) wb += s_wsum[b][w];
        const BlockOut& o = p.out[b];
        if (last_tile && threadIdx.x == 0) {  // chain totals: offsets[n], nnz, n_roots
            uint64_t tot = wb;
            for (int w = 0; w < kWarps; ++w) tot += s_wsum[b][w];
            o.offsets[n] = (int64_t)tot;
            *o.nnz_dev = (int64_t)tot;
            *o.n_roots_dev = n;
        }
        // block b's output j of this warp (warp-flat index fb + j) goes to global index wb + j
        const int64_t adj = (int64_t)wb - (int64_t)fb;
        if (lane < 3) wptr[b * 4 + lane] = (uint64_t)(lane == 0 ? (uintptr_t)(o.nbr + adj)
                                                       : lane == 1 ? (uintptr_t)(o.eid + adj) : (uintptr_t)(o.dt + adj));
        const uint32_t x = inc[b * 32 + lane];
        const uint32_t ex = __shfl_up_sync(kFull, x, 1);
        if (valid) o.offsets[i] = (int64_t)(wb + (lane ? ex : 0u));
        fb += __shfl_sync(kFull, x, 31);
    }
    __syncwarp();

    const int64_t warp_root0 = i - lane;  // global index of this warp's first root
    // flat copy over all snapshot blocks of the warp, 32 outputs per step: the windows starting in
    // the step's range set one bit each (one OR-reduction), so output o's window is found with a
    // popc -- h = (windows starting <= o) - 1 -- instead of a search
    const uint32_t total = flat;
    const uint32_t lemask = lanemask_lt() | (1u << lane);
    uint32_t hbase = 0;  // windows starting before o0
    constexpr int kCopyUnroll = STRATEGY == TGL_MOST_RECENT ? TGL_COPY_UNROLL : TGL_COPY_UNROLL_UNI;  // outputs in flight per lane
    for (uint32_t o0 = 0; o0 < total; o0 += 32 * kCopyUnroll) {
        uint32_t pos[kCopyUnroll], info[kCopyUnroll], oo[kCopyUnroll];
        bool act[kCopyUnroll];
#pragma unroll
        for (int u = 0; u < kCopyUnroll; ++u) {
            const uint32_t c0 = o0 + 32u * u;
            const uint32_t hl = hbase + lane;
            uint32_t bit = 0;
            if (hl < nseg) {
                const uint32_t st = (seg[hl].x >> 9) - c0;
                bit = st < 32u ? 1u << st : 0u;
            }
            const uint32_t heads = __reduce_or_sync(kFull, bit);
            const uint32_t o = c0 + (uint32_t)lane;
            act[u] = o < total;
            const uint32_t h = hbase + __popc(heads & lemask) - 1u;
            hbase += __popc(heads);
            TGL_CHECK(!act[u] || h < nseg);
            const uint2 sg = seg[act[u] ? h : 0u];
            const uint32_t q = o - (sg.x >> 9);
            info[u] = sg.x;
            oo[u] = o;
            if (VALID) {  // R#28: the window kernel's explicit selection
                const uint32_t b = (sg.x >> 5) & 15u, r = sg.x & 31u;
                pos[u] = act[u] ? p.vpicks[((size_t)b * p.roots_cap + (size_t)(warp_root0 + r)) * k + q] : 0u;
            } else if (STRATEGY == TGL_MOST_RECENT) {
                pos[u] = sg.y + q;
            } else {
                pos[u] = act[u] ? sg.y + picks[o] : 0u;
            }
        }
        int4 rec[kCopyUnroll];
#pragma unroll
        for (int u = 0; u < kCopyUnroll; ++u) {
            if (act[u]) {
                if (PK == 1) {
                    TGL_CHECK(pos[u] < p.n_stored);
                    const uint2 v = ld_rand_v2(reinterpret_cast<const uint2*>(p.recs) + pos[u]);
                    const uint64_t w = ((uint64_t)v.y << 32) | v.x;
                    const uint32_t c = (uint32_t)(w >> p.bn) & ((1u << p.bc) - 1u);
                    TGL_CHECK(c < (uint32_t)kMaxCodes);
                    rec[u] = make_int4(__float_as_int(s_tv[c]), (int32_t)(uint32_t)(w & ((1ull << p.bn) - 1ull)),
                                       s_te[c] + (int32_t)(uint32_t)(w >> (p.bn + p.bc)), 0);
                } else if (PK == 2) {  // integer times: ts = (float)time, exact below 2^24
                    TGL_CHECK(pos[u] < p.n_stored);
                    const uint2 v = STRATEGY == TGL_MOST_RECENT
                                        ? ld_rand_v2(reinterpret_cast<const uint2*>(p.recs) + pos[u])
                                        : ld_rand_v2_64(reinterpret_cast<const uint2*>(p.recs) + pos[u]);
                    const uint64_t w = ((uint64_t)v.y << 32) | v.x;
                    const uint32_t be = p.bc, sh = p.bn + p.bc;
                    rec[u] = make_int4(__float_as_int((float)(uint32_t)(w >> sh)),
                                       (int32_t)(uint32_t)(w & ((1ull << p.bn) - 1ull)),
                                       p.ebase0 + (int32_t)(uint32_t)((w >> p.bn) & ((1ull << be) - 1ull)), 0);
                } else if (p.recs) {
                    TGL_CHECK(pos[u] < p.n_stored);
                    rec[u] = ld_rec16<STRATEGY == TGL_MOST_RECENT && !VALID>(p.recs + pos[u]);
                } else {
                    rec[u] = make_int4(__float_as_int(__ldg(p.ts + pos[u])), __ldg(p.nbr + pos[u]),
                                       __ldg(p.eid + pos[u]), 0);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kCopyUnroll; ++u) {
            if (!act[u]) continue;
            const uint32_t b = (info[u] >> 5) & 15u, r = info[u] & 31u;
            const ulonglong2 pne = *reinterpret_cast<const ulonglong2*>(wptr + b * 4);
            float* dtp = reinterpret_cast<float*>(wptr[b * 4 + 2]);
            const float tv = __int_as_float(rec[u].x);
            const float tr = troot[r];
            // global-space stores (the pointers come from shared memory, so plain C++ stores compile
            // to generic ST.E; measured neutral on C4 / C5, kept for the SASS)
            st_global_u32(reinterpret_cast<int32_t*>(pne.x) + oo[u], (uint32_t)rec[u].y);
            st_global_u32(reinterpret_cast<int32_t*>(pne.y) + oo[u], (uint32_t)rec[u].z);
            st_global_u32(dtp + oo[u], __float_as_uint(__fsub_rn(tr, tv)));
            if (EXTRA) {
                const BlockOut& o = p.out[b];
                const uint64_t oi = (uint64_t)((reinterpret_cast<int32_t*>(pne.x) + oo[u]) - o.nbr);
                const uint32_t q = oo[u] - (info[u] >> 9);
                if (o.ts_edge) o.ts_edge[oi] = tv;
                if (o.child_key) o.child_key[oi] = rkey[r] * (uint64_t)k + q;
                if (o.child_t) o.child_t[oi] = tr;  // R#23: hop roots carry the root time
                if (o.child_lo)  // children inherit the window's lower bound (R#3)
                    o.child_lo[oi] = p.layer == 0 ? __fsub_rn(tr, __fmul_rn((float)(b + 1), p.snapshot_len))
                                                  : p.root_lo[warp_root0 + r];
            }
        }
        if (GATHER) {
#pragma unroll
            for (int u = 0; u < kCopyUnroll; ++u) {
                int64_t gi = 0;
                if (act[u]) {
                    const uint32_t b = (info[u] >> 5) & 15u;
                    gi = (int64_t)((reinterpret_cast<int32_t*>(wptr[b * 4]) + oo[u]) - p.out[b].nbr);
                }
                fused_gather_rows(p, act[u], gi, rec[u].y, rec[u].z, lane);
            }
        }
    }
}

// ---------------------------------------------------------------------------- K9 dedup (R#27)
// Distinct (node, hop time) pairs of a block in order of first appearance (SPEC's MFG node lists):
//   D1 insert: open addressing over 64-bit keys (node << 32 | time bits); the SLOT a key lands in
//      depends on the schedule, but atomicMin records the smallest output index per key, so
//   D2 flag: output i is a first occurrence iff it is its key's minimum -- deterministic; an
//      exclusive scan of the flags numbers the distinct pairs in first-appearance order;
//   D3 emit: src_index[i] = number of its key's first occurrence; firsts write the unique lists
//      (node, time, and the first occurrence's child key for the next layer's RNG, R#7).
__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ int64_t dev_count(const int64_t* n_dev, int64_t cap) {
    const int64_t m = *n_dev;
    return m < cap ? (m > 0 ? m : 0) : cap;
}

__global__ void dedup_insert_kernel(const int32_t* __restrict__ nbr, const float* __restrict__ t_hop,
                                    const int64_t* __restrict__ n_dev, int64_t cap, unsigned long long* hkeys,
                                    unsigned int* hfirst, uint64_t mask, uint32_t* __restrict__ slot_of) {
    const int64_t n = dev_count(n_dev, cap);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key =
            ((unsigned long long)(uint32_t)nbr[i] << 32) | (unsigned long long)__float_as_uint(t_hop[i]);
        uint64_t h = mix64(key) & mask;
        while (true) {
            const unsigned long long prev = atomicCAS(hkeys + h, ~0ull, key);
            if (prev == ~0ull || prev == key) break;
            h = (h + 1) & mask;
        }
        atomicMin(hfirst + h, (unsigned int)i);
        slot_of[i] = (uint32_t)h;
    }
}

__global__ void dedup_flag_kernel(const int64_t* __restrict__ n_dev, int64_t cap, const unsigned int* hfirst,
                                  const uint32_t* __restrict__ slot_of, uint32_t* __restrict__ flag) {
    const int64_t n = dev_count(n_dev, cap);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = i < n ? (hfirst[slot_of[i]] == (unsigned int)i ? 1u : 0u) : 0u;
}

__global__ void dedup_emit_kernel(const int32_t* __restrict__ nbr, const float* __restrict__ t_hop,
                                  const uint64_t* __restrict__ child_key, const int64_t* __restrict__ n_dev,
                                  int64_t cap, const unsigned int* hfirst, const uint32_t* __restrict__ slot_of,
                                  const uint32_t* __restrict__ flag, const uint32_t* __restrict__ uid,
                                  tgl_dedup_block o, uint64_t* __restrict__ uniq_key) {
    const int64_t n = dev_count(n_dev, cap);
    if (blockIdx.x == 0 && threadIdx.x == 0) *o.n_uniq_dev = n > 0 ? (int64_t)uid[n - 1] + flag[n - 1] : 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t u = uid[hfirst[slot_of[i]]];
        o.src_index[i] = (int32_t)u;
        if (flag[i]) {
            o.uniq_node[u] = nbr[i];
            o.uniq_ts[u] = t_hop[i];
            if (uniq_key) uniq_key[u] = child_key[i];
        }
    }
}

// the graph's arrays and aux structures in the kernel parameters.  The validity path (R#28) reads
// neither codec structure: with the codec its node records are the plain indptr + ts search and
// packed slot records fall back to the separate arrays
static void set_graph(SampleParams& sp, const tgl_tcsr* g, bool use_recs, bool use_index, bool validity) {
    sp.indptr = g->indptr;
    sp.nbr = g->nbr;
    sp.ts = g->ts;
    sp.eid = g->eid;
    const bool codec = use_recs && g->n_codes > 0;
    sp.recs = use_recs && !(validity && g->packed) ? static_cast<const SlotRec*>(g->recs) : nullptr;
    sp.nodes = use_recs && !(validity && codec) ? static_cast<const int4*>(g->nodes) : nullptr;
    if (codec && !validity) {
        const TimeDict* d = static_cast<const TimeDict*>(g->dict);
        sp.codes = g->codes;
        sp.tval = d->value;
        sp.tebase = d->eid_base;
        sp.packed = g->packed;
        sp.bn = (uint32_t)g->bits_nbr;
        sp.bc = (uint32_t)g->bits_code;
    } else if (use_recs && g->packed == 2 && !validity) {
        sp.packed = 2;
        sp.bn = (uint32_t)g->bits_nbr;
        sp.bc = (uint32_t)g->bits_code;
        sp.ebase0 = g->eid_base0;
    }
    sp.n_stored = (uint32_t)g->n_stored;
    sp.n_levels = use_index && g->index ? g->n_levels : 0;
    for (int q = 1; q <= sp.n_levels; ++q) sp.lvl[q] = g->index + g->level_off[q];
    sp.n_nodes = g->n_nodes;
    sp.node_lo = g->node_lo;
}

static bool picks_fit_smem(int nsb, int k) { return (size_t)nsb * k * 32 * 4 <= kPicksSmemPerWarp; }

struct Launch {
    int layer, chain, nsb;
    int64_t roots_cap, tiles_cap;
    uint32_t *cuts, *tile_tot;
    uint64_t* super_tot;
    int64_t supers_cap;
    uint64_t* hyper_tot;
    int64_t hypers_cap;
    uint32_t* picks;  // global picks or null
    uint32_t *vpicks, *vtake;  // R#28 explicit selection (edge validity) or null
};

struct SamplePlan {
    int L = 0, S = 0;
    int64_t roots_cap[64], edges_cap[64];
    Launch launches[1 + 63 * TGL_MAX_SNAPSHOTS];
    int n_launch = 0;
    size_t memset_from = 0, memset_bytes = 0;
    uint64_t* child_key[64][TGL_MAX_SNAPSHOTS];
    float* child_lo[64][TGL_MAX_SNAPSHOTS];
    float* child_t[64][TGL_MAX_SNAPSHOTS];
    uint64_t* uniq_key[64][TGL_MAX_SNAPSHOTS];  // dedup: first occurrence's child key per distinct pair
    // dedup scratch (one block at a time): hash keys / first index, slot per output, flags, ids
    unsigned long long* hkeys = nullptr;
    unsigned int* hfirst = nullptr;
    uint64_t hsize = 0;
    uint32_t *slot_of = nullptr, *flag = nullptr, *uid = nullptr;
    uint64_t* scan_partial = nullptr;
    size_t bytes = 0;
};

static int plan_sample(int64_t n_roots, int L, const int32_t* fanouts, int S, int strategy, float snapshot_len,
                       bool dedup, bool hop_root, bool validity, void* ws, SamplePlan& P) {
    if (L < 1 || L > 64 || S < 1 || S > TGL_MAX_SNAPSHOTS || n_roots < 0 || !fanouts) return TGL_EINVAL;
    if (!(snapshot_len > 0.0f)) return TGL_EINVAL;               // NaN or <= 0
    if (S > 1 && !std::isfinite(snapshot_len)) return TGL_EINVAL;  // +inf only for one snapshot
    if (strategy != TGL_MOST_RECENT && strategy != TGL_UNIFORM) return TGL_EINVAL;
    P.L = L;
    P.S = S;
    int64_t r = n_roots;
    for (int l = 0; l < L; ++l) {
        const int k = fanouts[l];
        if (k < 1 || k > TGL_MAX_FANOUT) return TGL_EINVAL;
        if (r > (int64_t)1 << 40) return TGL_EINVAL;
        P.roots_cap[l] = r;
        P.edges_cap[l] = r * k;
        r = r * k;
    }
    Carve c(ws);
    P.n_launch = 0;
    auto add = [&](int layer, int chain, int nsb) {
        Launch& la = P.launches[P.n_launch++];
        la.layer = layer;
        la.chain = chain;
        la.nsb = nsb;
        la.roots_cap = std::max<int64_t>(1, P.roots_cap[layer]);
        la.tiles_cap = (la.roots_cap + kTile - 1) / kTile;
        la.cuts = c.take<uint32_t>((size_t)(nsb + 1) * la.roots_cap);
        la.tile_tot = c.take<uint32_t>((size_t)nsb * la.tiles_cap);
        la.supers_cap = (la.tiles_cap + (1 << kSuperShift) - 1) >> kSuperShift;
        la.hypers_cap = (la.supers_cap + (1 << kSuperShift) - 1) >> kSuperShift;
        la.picks = nullptr;
        if (strategy == TGL_UNIFORM && !picks_fit_smem(nsb, fanouts[layer]))
            la.picks = c.take<uint32_t>((size_t)la.tiles_cap * kTile * nsb * fanouts[layer]);
        la.vpicks = validity ? c.take<uint32_t>((size_t)nsb * la.roots_cap * fanouts[layer]) : nullptr;
        la.vtake = validity ? c.take<uint32_t>((size_t)nsb * la.roots_cap) : nullptr;
    };
    add(0, 0, S);
    for (int l = 1; l < L; ++l)
        for (int s = 0; s < S; ++s) add(l, s, 1);
    // super totals of every chain together: one contiguous region, one memset per call
    P.memset_from = c.bytes();
    for (int j = 0; j < P.n_launch; ++j)
        P.launches[j].super_tot = c.take<uint64_t>((size_t)P.launches[j].nsb * P.launches[j].supers_cap);
    for (int j = 0; j < P.n_launch; ++j)
        P.launches[j].hyper_tot = c.take<uint64_t>((size_t)P.launches[j].nsb * P.launches[j].hypers_cap);
    P.memset_bytes = c.bytes() - P.memset_from;
    const bool need_lo = L > 1 && std::isfinite(snapshot_len);
    if (dedup && need_lo) return TGL_EINVAL;  // R#27: windows with inherited finite bounds would merge
    for (int l = 0; l < L; ++l)
        for (int s = 0; s < S; ++s) {
            const bool inner = l < L - 1;
            P.child_key[l][s] = inner && strategy == TGL_UNIFORM ? c.take<uint64_t>((size_t)P.edges_cap[l]) : nullptr;
            P.child_lo[l][s] = inner && need_lo ? c.take<float>((size_t)P.edges_cap[l]) : nullptr;
            // hop-root times under TGL_HOP_ROOT_TIME (the last layer's only for dedup keys)
            P.child_t[l][s] = inner || (dedup && hop_root) ? c.take<float>((size_t)P.edges_cap[l]) : nullptr;
            P.uniq_key[l][s] = inner && dedup && strategy == TGL_UNIFORM ? c.take<uint64_t>((size_t)P.edges_cap[l])
                                                                         : nullptr;
        }
    if (dedup) {
        int64_t emax = 1;
        for (int l = 0; l < L; ++l) emax = std::max<int64_t>(emax, P.edges_cap[l]);
        uint64_t h = 64;
        while (h < 2 * (uint64_t)emax) h <<= 1;
        P.hsize = h;
        P.hkeys = c.take<unsigned long long>(h);
        P.hfirst = c.take<unsigned int>(h);
        P.slot_of = c.take<uint32_t>((size_t)emax);
        P.flag = c.take<uint32_t>((size_t)emax);
        P.uid = c.take<uint32_t>((size_t)emax);
        P.scan_partial = c.take<uint64_t>(scan_workspace_bytes(emax) / sizeof(uint64_t) + 1);
    }
    P.bytes = c.bytes();
    return TGL_OK;
}

template <int STRATEGY, bool VALID, int OUTX, bool PSMEM, int PK>
static void launch_copy_pk(const SampleParams& sp, int64_t grid, size_t smem, cudaStream_t st) {
    if (PK == 1) smem += 256 * (sizeof(float) + sizeof(int32_t));  // the codec's dictionaries
    if (smem + 1024 > 48 * 1024)  // the dynamic part plus ~640 B of static shared memory
        cudaFuncSetAttribute(copy_kernel<STRATEGY, VALID, OUTX, PSMEM, PK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    // programmatic dependent launch (PDL): the copy grid is launched while the window grid's last
    // CTAs finish and waits in griddepcontrol.wait -- hides the launch gap between the two
    static const bool no_pdl = getenv("TGL_NO_PDL") != nullptr;  // A/B knob
    if (no_pdl) {
        copy_kernel<STRATEGY, VALID, OUTX, PSMEM, PK><<<(unsigned)grid, kTile, smem, st>>>(sp);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kTile);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, copy_kernel<STRATEGY, VALID, OUTX, PSMEM, PK>, sp);
}

// packed records exist only with the codec, which the validity path never uses
template <int STRATEGY, bool VALID, int OUTX, bool PSMEM>
static void launch_copy_ps(const SampleParams& sp, int64_t grid, size_t smem, cudaStream_t st) {
    if (!VALID && sp.packed == 1)
        launch_copy_pk<STRATEGY, VALID, OUTX, PSMEM, VALID ? 0 : 1>(sp, grid, smem, st);
    else if (!VALID && sp.packed == 2)
        launch_copy_pk<STRATEGY, VALID, OUTX, PSMEM, VALID ? 0 : 2>(sp, grid, smem, st);
    else
        launch_copy_pk<STRATEGY, VALID, OUTX, PSMEM, 0>(sp, grid, smem, st);
}

template <int STRATEGY, bool VALID, int OUTX>
static void launch_copy(const SampleParams& sp, int64_t grid, size_t smem, cudaStream_t st) {
    if (STRATEGY == TGL_UNIFORM && sp.picks_global == nullptr)
        launch_copy_ps<STRATEGY, VALID, OUTX, true>(sp, grid, smem, st);
    else
        launch_copy_ps<STRATEGY, VALID, OUTX, false>(sp, grid, smem, st);
}

// EXTRA: the chain writes per-output data for a following layer or the dedup (ts_edge, child
// key / time / lower bound); the last layer's copy carries none of it
template <int STRATEGY, bool VALID>
static int launch_pair(const SampleParams& sp, int64_t grid, size_t smem, cudaStream_t st) {
    if (!VALID && sp.codes)
        window_kernel<STRATEGY, VALID, !VALID><<<(unsigned)grid, kTile, 0, st>>>(sp);
    else
        window_kernel<STRATEGY, VALID, false><<<(unsigned)grid, kTile, 0, st>>>(sp);
    bool extra = false;
    for (int b = 0; b < sp.nsb; ++b)
        extra |= sp.out[b].ts_edge || sp.out[b].child_key || sp.out[b].child_t || sp.out[b].child_lo;
    if (extra)
        launch_copy<STRATEGY, VALID, 1>(sp, grid, smem, st);
    else if (!VALID && sp.fg.n > 0)  // fused gather: last-layer chains only (never with extra data)
        launch_copy<STRATEGY, false, 2>(sp, grid, smem, st);
    else
        launch_copy<STRATEGY, VALID, 0>(sp, grid, smem, st);
    return cudaGetLastError() == cudaSuccess ? TGL_OK : TGL_ECUDA;
}

// the validity path (R#28) is a separate instantiation: the default kernels carry none of it
template <int STRATEGY>
static int launch_chain(const SampleParams& sp, int64_t grid, size_t smem, cudaStream_t st) {
    return sp.valid ? launch_pair<STRATEGY, true>(sp, grid, smem, st) : launch_pair<STRATEGY, false>(sp, grid, smem, st);
}

// Layer l >= 1 chains of different snapshots are independent (chain (l, s) reads only block
// (l-1, s), Alg. 1 L227 / R#3, and each chain has its own workspace slice): with S > 1 they run
// on S forked streams joined back by events, so one snapshot's tail overlaps the next one's
// kernels.  Library-owned, created once per (thread, device); not used while the caller's
// stream is being captured into a CUDA graph (the sequential order is captured instead).
struct ForkStreams {
    int dev = -1;
    cudaStream_t side[TGL_MAX_SNAPSHOTS] = {};
    cudaEvent_t fork = nullptr, join[TGL_MAX_SNAPSHOTS] = {};
};

static ForkStreams* fork_streams(int S) {
    static thread_local ForkStreams F[16];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
    ForkStreams& f = F[dev];
    if (f.dev != dev) {
        if (cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        f.dev = dev;
    }
    for (int s = 0; s < S; ++s)
        if (!f.side[s] && (cudaStreamCreateWithFlags(&f.side[s], cudaStreamNonBlocking) != cudaSuccess ||
                           cudaEventCreateWithFlags(&f.join[s], cudaEventDisableTiming) != cudaSuccess))
            return nullptr;
    return &f;
}

// ---------------------------------------------------------------------------- one chain, explicit roots
// The owner side of the node-sharded exchange (sharded.cu): one chain -- layer `layer`, all nsb
// snapshot blocks of a layer-0 root (snap0 = 0) or snapshot snap0's block at l >= 1 -- over roots
// received from other ranks, each with its explicit key (R#7) and, at l >= 1, its inherited lower
// bound (R#3): the same two kernels and the same Philox counters as tgl_sample, so the blocks are
// those the replicated mode writes for these roots.
static Launch plan_chain(int64_t n, int nsb, int k, int strategy, void* ws, size_t* bytes) {
    Carve c(ws);
    Launch la;
    memset(&la, 0, sizeof(la));
    la.nsb = nsb;
    la.roots_cap = std::max<int64_t>(1, n);
    la.tiles_cap = (la.roots_cap + kTile - 1) / kTile;
    la.cuts = c.take<uint32_t>((size_t)(nsb + 1) * la.roots_cap);
    la.tile_tot = c.take<uint32_t>((size_t)nsb * la.tiles_cap);
    la.supers_cap = (la.tiles_cap + (1 << kSuperShift) - 1) >> kSuperShift;
    la.hypers_cap = (la.supers_cap + (1 << kSuperShift) - 1) >> kSuperShift;
    if (strategy == TGL_UNIFORM && !picks_fit_smem(nsb, k))
        la.picks = c.take<uint32_t>((size_t)la.tiles_cap * kTile * nsb * k);
    la.super_tot = c.take<uint64_t>((size_t)nsb * la.supers_cap);
    la.hyper_tot = c.take<uint64_t>((size_t)nsb * la.hypers_cap);
    if (bytes) *bytes = c.bytes();
    return la;
}

size_t chain_workspace_bytes(int64_t n, int nsb, int k, int strategy) {
    size_t b = 0;
    plan_chain(n, nsb, k, strategy, nullptr, &b);
    return b;
}

int sample_chain(const tgl_tcsr* g, int layer, int snap0, int nsb, const int32_t* rn, const float* rt,
                 const uint64_t* rk, const float* rlo, int64_t n, int k, int strategy, float t_s, uint64_t seed,
                 const ChainOut* outs, void* ws, size_t ws_bytes, cudaStream_t st) {
    if (nsb < 1 || nsb > TGL_MAX_SNAPSHOTS || k < 1 || k > TGL_MAX_FANOUT || n < 0 || !ws) return TGL_EINVAL;
    size_t need = 0;
    const Launch la = plan_chain(n, nsb, k, strategy, ws, &need);
    if (ws_bytes < need) return TGL_EWORKSPACE;
    if (la.tiles_cap > (1 << kSuperShift) &&
        cudaMemsetAsync(la.super_tot, 0,
                        (size_t)(reinterpret_cast<char*>(la.hyper_tot + (size_t)nsb * la.hypers_cap) -
                                 reinterpret_cast<char*>(la.super_tot)),
                        st) != cudaSuccess)
        return TGL_ECUDA;
    SampleParams sp;
    memset(&sp, 0, sizeof(sp));
    set_graph(sp, g, g->recs != nullptr, g->index != nullptr, false);
    sp.root_node = rn;
    sp.root_ts = rt;
    sp.root_key = rk;
    sp.root_lo = layer > 0 ? rlo : nullptr;
    sp.n_roots = n;
    sp.layer = layer;
    sp.nsb = nsb;
    sp.snap0 = snap0;
    sp.k = k;
    sp.snapshot_len = t_s;
    sp.seed_lo = (uint32_t)seed;
    sp.seed_hi = (uint32_t)(seed >> 32);
    sp.cuts = la.cuts;
    sp.tile_tot = la.tile_tot;
    sp.super_tot = la.super_tot;
    sp.supers_cap = la.supers_cap;
    sp.hyper_tot = la.hyper_tot;
    sp.hypers_cap = la.hypers_cap;
    sp.roots_cap = la.roots_cap;
    sp.tiles_cap = la.tiles_cap;
    sp.picks_global = la.picks;
    sp.err = g->err_dev;
    for (int b = 0; b < nsb; ++b) {
        BlockOut& bo = sp.out[b];
        bo.offsets = outs[b].offsets;
        bo.nbr = outs[b].nbr;
        bo.eid = outs[b].eid;
        bo.dt = outs[b].dt;
        bo.ts_edge = outs[b].ts_edge;
        bo.n_roots_dev = outs[b].n_roots_dev;
        bo.nnz_dev = outs[b].nnz_dev;
    }
    const int64_t tiles = std::max<int64_t>(1, (n + kTile - 1) / kTile);
    const size_t smem = (size_t)kWarps * copy_warp_words(nsb, k, strategy == TGL_UNIFORM && la.picks == nullptr) * 4;
    return strategy == TGL_UNIFORM ? launch_chain<TGL_UNIFORM>(sp, tiles, smem, st)
                                   : launch_chain<TGL_MOST_RECENT>(sp, tiles, smem, st);
}

}  // namespace tgl

using namespace tgl;

extern "C" int tgl_sample_capacity(int64_t n_roots, int32_t n_layers, const int32_t* fanouts, int32_t n_snapshots,
                                   tgl_strategy strategy, float snapshot_len, int64_t* roots_cap, int64_t* edges_cap,
                                   size_t* ws_bytes) {
    static thread_local SamplePlan P;
    int rc = plan_sample(n_roots, n_layers, fanouts, n_snapshots, (int)strategy, snapshot_len, false, false, false,
                         nullptr, P);
    if (rc) return rc;
    for (int l = 0; l < n_layers; ++l) {
        if (roots_cap) roots_cap[l] = P.roots_cap[l];
        if (edges_cap) edges_cap[l] = P.edges_cap[l];
    }
    if (ws_bytes) *ws_bytes = P.bytes;
    return TGL_OK;
}

static int sample_impl(const tgl_tcsr* g, const int32_t* roots, const float* root_ts, const uint64_t* root_keys,
                       int64_t n_roots, int32_t n_layers, const int32_t* fanouts, tgl_strategy strategy,
                       int32_t n_snapshots, float snapshot_len, uint64_t seed, uint64_t root_key_base,
                       const tgl_sample_options* opts, tgl_block* out, const tgl_dedup_block* dd,
                       void* workspace, size_t ws_bytes, void* stream) {
    NvtxRange nvtx_("tgl_sample");
    if (!g || !out || !workspace) return TGL_EINVAL;
    tgl_sample_options o;
    memset(&o, 0, sizeof(o));
    if (opts) o = *opts;
    if (o.hop_time != TGL_HOP_EDGE_TIME && o.hop_time != TGL_HOP_ROOT_TIME) return TGL_EINVAL;
    if (o.replacement != 0 && (o.replacement != 1 || strategy != TGL_UNIFORM)) return TGL_EINVAL;
    if (o.dedup != 0 && (o.dedup != 1 || !dd)) return TGL_EINVAL;
    for (int q = 0; q < 5; ++q)
        if (o.reserved[q]) return TGL_EINVAL;
    const bool hop_root = o.hop_time == TGL_HOP_ROOT_TIME;
    const bool dedup = o.dedup == 1;
    FusedGather fg;
    memset(&fg, 0, sizeof(fg));
    if (o.gather) {  // fused gather of the last layer's block
        const tgl_fused_gather& G = *o.gather;
        if (G.n_tables < 1 || G.n_tables > TGL_MAX_FUSED_GATHER || n_snapshots != 1 || dedup || o.edge_valid)
            return TGL_EINVAL;
        fg.n = G.n_tables;
        for (int j = 0; j < G.n_tables; ++j) {
            const tgl_fused_table& t = G.tables[j];
            if (!t.out || t.row_bytes <= 0 || (t.row_bytes & 3) || t.n_rows < 0 || (t.n_rows > 0 && !t.table) ||
                (t.by_edge != 0 && t.by_edge != 1))
                return TGL_EINVAL;
            const bool v16 = (t.row_bytes % 16) == 0 && ((uintptr_t)t.table % 16) == 0 && ((uintptr_t)t.out % 16) == 0;
            fg.t[j] = FusedTable{t.table, t.out, t.n_rows, v16 ? (uint32_t)(t.row_bytes / 16) : 0u,
                                 (uint32_t)(t.row_bytes / 4), t.by_edge};
        }
    }
    if (n_roots > 0 && (!roots || !root_ts)) return TGL_EINVAL;
    static thread_local SamplePlan P;
    int rc = plan_sample(n_roots, n_layers, fanouts, n_snapshots, (int)strategy, snapshot_len, dedup, hop_root,
                         o.edge_valid != nullptr, workspace, P);
    if (rc) return rc;
    if (ws_bytes < P.bytes) return TGL_EWORKSPACE;
    rc = check_device();
    if (rc) return rc;
    const int L = n_layers, S = n_snapshots;
    for (int l = 0; l < L; ++l)
        for (int s = 0; s < S; ++s) {
            const tgl_block& b = out[l * S + s];
            if (!b.offsets || !b.nbr || !b.eid || !b.dt || !b.n_roots_dev || !b.nnz_dev) return TGL_EINVAL;
            if ((l < L - 1 || (dedup && !hop_root)) && !b.ts_edge) return TGL_EINVAL;
            if (b.cap_roots < P.roots_cap[l] || b.cap_edges < P.edges_cap[l]) return TGL_ECAPACITY;
            if (dedup) {
                const tgl_dedup_block& d = dd[l * S + s];
                if (!d.src_index || !d.uniq_node || !d.uniq_ts || !d.n_uniq_dev) return TGL_EINVAL;
                if (d.cap < P.edges_cap[l]) return TGL_ECAPACITY;
            }
        }
    cudaStream_t st = (cudaStream_t)stream;
    // super totals are read only for super tiles BEFORE a copy CTA's own: a call whose chains all
    // fit one super tile (<= 64 tiles: per-batch calls) never reads them, so needs no zeroing
    bool need_zero = false;
    for (int j = 0; j < P.n_launch; ++j) need_zero |= P.launches[j].tiles_cap > (1 << kSuperShift);
    if (need_zero &&
        cudaMemsetAsync(static_cast<char*>(workspace) + P.memset_from, 0, P.memset_bytes, st) != cudaSuccess)
        return TGL_ECUDA;
    // A/B knobs (tools/sweep.py), read once per process: TGL_NO_RECS / TGL_NO_INDEX run the same
    // kernels over the plain T-CSR arrays
    static const bool no_recs = getenv("TGL_NO_RECS") != nullptr;
    static const bool no_index = getenv("TGL_NO_INDEX") != nullptr;
    const bool use_recs = g->recs && !no_recs;
    const bool use_index = g->index && g->n_levels > 0 && !no_index;
    static const bool no_fork = getenv("TGL_NO_FORK") != nullptr;  // A/B knob
    ForkStreams* fk = nullptr;
    if (S > 1 && L > 1 && !dedup && !no_fork) {  // dedup shares one scratch across chains: sequential
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone)
            fk = fork_streams(S);
    }
    for (int j = 0; j < P.n_launch; ++j) {
        const Launch& la = P.launches[j];
        const int l = la.layer, s = la.chain;
        if (fk && j == 1) {  // after layer 0: fork the snapshot chains
            if (cudaEventRecord(fk->fork, st) != cudaSuccess) return TGL_ECUDA;
            for (int q = 0; q < S; ++q)
                if (cudaStreamWaitEvent(fk->side[q], fk->fork, 0) != cudaSuccess) return TGL_ECUDA;
        }
        cudaStream_t cst = fk && l > 0 ? fk->side[s] : st;
        SampleParams sp;
        memset(&sp, 0, sizeof(sp));
        set_graph(sp, g, use_recs, use_index, o.edge_valid != nullptr);
        if (l == 0) {
            sp.root_node = roots;
            sp.root_ts = root_ts;
            sp.root_key = root_keys;
            sp.n_roots = n_roots;
        } else {
            const tgl_block& par = out[(l - 1) * S + s];
            if (dedup) {  // R#27: the previous block's distinct (node, time) pairs
                const tgl_dedup_block& pd = dd[(l - 1) * S + s];
                sp.root_node = pd.uniq_node;
                sp.root_ts = pd.uniq_ts;
                sp.root_key = P.uniq_key[l - 1][s];
                sp.root_lo = nullptr;
                sp.n_roots_dev_in = pd.n_uniq_dev;
            } else {
                sp.root_node = par.nbr;
                sp.root_ts = hop_root ? P.child_t[l - 1][s] : par.ts_edge;
                sp.root_key = P.child_key[l - 1][s];
                sp.root_lo = P.child_lo[l - 1][s];
                sp.n_roots_dev_in = par.nnz_dev;
            }
            sp.n_roots = P.roots_cap[l];
        }
        sp.root_key_base = root_key_base;
        sp.layer = l;
        sp.nsb = la.nsb;
        sp.snap0 = s;
        sp.k = fanouts[l];
        sp.replacement = o.replacement;
        sp.valid = o.edge_valid;
        sp.vpicks = la.vpicks;
        sp.vtake = la.vtake;
        sp.snapshot_len = snapshot_len;
        sp.seed_lo = (uint32_t)seed;
        sp.seed_hi = (uint32_t)(seed >> 32);
        sp.cuts = la.cuts;
        sp.tile_tot = la.tile_tot;
        sp.super_tot = la.super_tot;
        sp.supers_cap = la.supers_cap;
        sp.hyper_tot = la.hyper_tot;
        sp.hypers_cap = la.hypers_cap;
        sp.roots_cap = la.roots_cap;
        sp.tiles_cap = la.tiles_cap;
        sp.picks_global = la.picks;
        sp.err = g->err_dev;
        if (l == L - 1) sp.fg = fg;  // the fused gather rides on the last layer's copy kernel
        for (int b = 0; b < la.nsb; ++b) {
            const int bs = l == 0 ? b : s;  // snapshot of output b
            const tgl_block& ob = out[l * S + bs];
            BlockOut& bo = sp.out[b];
            bo.offsets = ob.offsets;
            bo.nbr = ob.nbr;
            bo.eid = ob.eid;
            bo.dt = ob.dt;
            bo.ts_edge = ob.ts_edge;
            bo.child_key = l < L - 1 ? P.child_key[l][bs] : nullptr;
            bo.child_lo = l < L - 1 ? P.child_lo[l][bs] : nullptr;
            bo.child_t = hop_root ? P.child_t[l][bs] : nullptr;  // null for the last layer without dedup
            bo.n_roots_dev = ob.n_roots_dev;
            bo.nnz_dev = ob.nnz_dev;
        }
        const int64_t tiles = l == 0 ? std::max<int64_t>(1, (n_roots + kTile - 1) / kTile) : la.tiles_cap;
        const size_t smem =
            (size_t)kWarps * copy_warp_words(la.nsb, sp.k, strategy == TGL_UNIFORM && la.picks == nullptr) * 4;
        rc = strategy == TGL_UNIFORM ? launch_chain<TGL_UNIFORM>(sp, tiles, smem, cst)
                                     : launch_chain<TGL_MOST_RECENT>(sp, tiles, smem, cst);
        if (rc) return rc;
        if (dedup) {
            for (int b = 0; b < la.nsb; ++b) {
                const int bs = l == 0 ? b : s;
                const tgl_block& ob = out[l * S + bs];
                const float* t_hop = hop_root ? P.child_t[l][bs] : ob.ts_edge;
                const int64_t cap = P.edges_cap[l];
                const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((cap + 255) / 256, 148 * 8));
                if (cudaMemsetAsync(P.hkeys, 0xff, P.hsize * sizeof(unsigned long long), st) != cudaSuccess ||
                    cudaMemsetAsync(P.hfirst, 0xff, P.hsize * sizeof(unsigned int), st) != cudaSuccess)
                    return TGL_ECUDA;
                dedup_insert_kernel<<<blocks, 256, 0, st>>>(ob.nbr, t_hop, ob.nnz_dev, cap, P.hkeys, P.hfirst,
                                                            P.hsize - 1, P.slot_of);
                dedup_flag_kernel<<<blocks, 256, 0, st>>>(ob.nnz_dev, cap, P.hfirst, P.slot_of, P.flag);
                if (cuda_rc(exclusive_scan<uint32_t, uint32_t>(P.flag, P.uid, cap, (uint32_t*)nullptr, P.scan_partial,
                                                               st)))
                    return TGL_ECUDA;
                dedup_emit_kernel<<<blocks, 256, 0, st>>>(ob.nbr, t_hop, P.child_key[l][bs], ob.nnz_dev, cap, P.hfirst,
                                                          P.slot_of, P.flag, P.uid, dd[l * S + bs],
                                                          P.uniq_key[l][bs]);
                if (cudaGetLastError() != cudaSuccess) return TGL_ECUDA;
            }
        }
    }
    if (fk)  // join: the caller's stream waits for every snapshot chain
        for (int q = 0; q < S; ++q)
            if (cudaEventRecord(fk->join[q], fk->side[q]) != cudaSuccess || cudaStreamWaitEvent(st, fk->join[q], 0) != cudaSuccess)
                return TGL_ECUDA;
    return TGL_OK;
}

extern "C" int tgl_sample(const tgl_tcsr* g, const int32_t* roots, const float* root_ts, int64_t n_roots,
                          int32_t n_layers, const int32_t* fanouts, tgl_strategy strategy, int32_t n_snapshots,
                          float snapshot_len, uint64_t seed, uint64_t root_key_base, tgl_block* out, void* workspace,
                          size_t ws_bytes, void* stream) {
    return sample_impl(g, roots, root_ts, nullptr, n_roots, n_layers, fanouts, strategy, n_snapshots, snapshot_len,
                       seed, root_key_base, nullptr, out, nullptr, workspace, ws_bytes, stream);
}

extern "C" int tgl_sample_keyed(const tgl_tcsr* g, const int32_t* roots, const float* root_ts,
                                const uint64_t* root_keys, int64_t n_roots, int32_t n_layers, const int32_t* fanouts,
                                tgl_strategy strategy, int32_t n_snapshots, float snapshot_len, uint64_t seed,
                                tgl_block* out, void* workspace, size_t ws_bytes, void* stream) {
    if (n_roots > 0 && !root_keys) return TGL_EINVAL;
    return sample_impl(g, roots, root_ts, root_keys, n_roots, n_layers, fanouts, strategy, n_snapshots, snapshot_len,
                       seed, 0, nullptr, out, nullptr, workspace, ws_bytes, stream);
}

extern "C" int tgl_sample_ex(const tgl_tcsr* g, const int32_t* roots, const float* root_ts, const uint64_t* root_keys,
                             int64_t n_roots, int32_t n_layers, const int32_t* fanouts, tgl_strategy strategy,
                             int32_t n_snapshots, float snapshot_len, uint64_t seed, uint64_t root_key_base,
                             const tgl_sample_options* opts, tgl_block* out, const tgl_dedup_block* dedup,
                             void* workspace, size_t ws_bytes, void* stream) {
    return sample_impl(g, roots, root_ts, root_keys, n_roots, n_layers, fanouts, strategy, n_snapshots, snapshot_len,
                       seed, root_keys ? 0 : root_key_base, opts, out, dedup, workspace, ws_bytes, stream);
}

extern "C" int tgl_sample_capacity_ex(int64_t n_roots, int32_t n_layers, const int32_t* fanouts, int32_t n_snapshots,
                                      tgl_strategy strategy, float snapshot_len, const tgl_sample_options* opts,
                                      int64_t* roots_cap, int64_t* edges_cap, size_t* ws_bytes) {
    tgl_sample_options o;
    memset(&o, 0, sizeof(o));
    if (opts) o = *opts;
    static thread_local SamplePlan P;
    int rc = plan_sample(n_roots, n_layers, fanouts, n_snapshots, (int)strategy, snapshot_len, o.dedup == 1,
                         o.hop_time == TGL_HOP_ROOT_TIME, o.edge_valid != nullptr, nullptr, P);
    if (rc) return rc;
    for (int l = 0; l < n_layers; ++l) {
        if (roots_cap) roots_cap[l] = P.roots_cap[l];
        if (edges_cap) edges_cap[l] = P.edges_cap[l];
    }
    if (ws_bytes) *ws_bytes = P.bytes;
    return TGL_OK;
}
