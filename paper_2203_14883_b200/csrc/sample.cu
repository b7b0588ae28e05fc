// sample.cu -- the parallel temporal sampler of TGL (Alg. 1) on B200.
//
// One kernel launch per (layer, chain).  Layer 0 is a single chain covering all S dynamic
// snapshots of a root in one pass (the S+1 cuts of a root share its indptr pair and narrow
// each other's search range); a layer l >= 1 runs one chain per snapshot s whose roots are
// block (l-1, s)'s outputs (Alg. 1, R#3).
//
// A CTA owns a tile of 256 consecutive roots (tile index from an atomic ticket, so tiles start in
// order and the look-back below always waits on running or finished CTAs):
//   phase 1  one thread per root: indptr pair (16 B), S+1 cut searches by binary search over
//            the node's time-sorted list (Sec. 3.1 "Sampling", L260-L262: the stateless
//            replacement of the per-node pointers pt_0..pt_S), selection:
//              most_recent -> [max(a, b-k), b)           ("closest to the end pointer")
//              uniform     -> all of [a, b) if c <= k, else Floyd's k-subset with Philox4x32-10
//                             draws, sorted ascending (R#5, R#6)
//   phase 2  block scan of per-root counts + decoupled look-back across tiles (one chained
//            scan per snapshot) -> deterministic CSR offsets without a second pass (K5)
//   phase 3  the tile's outputs are copied as one flat range: thread o finds its root by a
//            binary search over the tile's inclusive counts in shared memory, so loads of
//            (nbr, eid, ts) and stores of (nbr, eid, dt[, ts_edge, child key, child lo]) are
//            coalesced and every lane is busy (a9, a10; K6 fused).
// dt = t_root (-) t_edge with __fsub_rn; window bounds with __fmul_rn / __fsub_rn (R#12).
// Everything strictly before the root: ts < U = t.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.cuh"

namespace tgl {

constexpr int kSampleThreads = 256;  // roots per tile
constexpr int kSampleWarps = kSampleThreads / 32;
constexpr int kCopyUnroll = 4;
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagPrefix = 2ull << 62, kValMask = (1ull << 62) - 1;
constexpr size_t kPicksSmemLimit = 64 * 1024;

struct BlockOut {
    int64_t* offsets;
    int32_t* nbr;
    int32_t* eid;
    float* dt;
    float* ts_edge;       // may be null
    uint64_t* child_key;  // may be null
    float* child_lo;      // may be null
    int64_t* n_roots_dev;
    int64_t* nnz_dev;
};

struct SampleParams {
    const int64_t* indptr;
    const int32_t* nbr;
    const float* ts;
    const int32_t* eid;
    int32_t n_nodes;
    const int32_t* root_node;
    const float* root_ts;
    const uint64_t* root_key;  // l >= 1 (uniform): parent layer's child keys; null at layer 0
    const float* root_lo;      // l >= 1: inherited lower bounds; null -> -inf
    uint64_t root_key_base;
    int64_t n_roots;                // layer 0: count; l >= 1: capacity
    const int64_t* n_roots_dev_in;  // l >= 1: device count (parent block's nnz)
    int32_t layer, nsb, snap0, k;
    float snapshot_len;
    uint32_t seed_lo, seed_hi;
    uint64_t* tile_state;  // [nsb][tiles_cap], zeroed before the launch
    uint32_t* tile_counter;
    int64_t tiles_cap;
    uint32_t* picks_global;  // null -> picks in shared memory
    int* err;
    BlockOut out[TGL_MAX_SNAPSHOTS];
};

// First slot p in [lo, hi) with ts[p] >= x (else hi): the cut of a window (R#2).
__device__ __forceinline__ uint32_t lower_bound_ts(const float* __restrict__ ts, uint32_t lo, uint32_t hi, float x) {
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(ts + mid) < x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// Block-wide exclusive scan (uint32 counts, uint64 totals).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total, uint32_t* sm /*[kSampleWarps+1]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < kSampleWarps ? sm[lane] : 0;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < kSampleWarps) sm[lane] = wi - w;
        if (lane == kSampleWarps - 1) sm[kSampleWarps] = wi;
    }
    __syncthreads();
    const uint32_t r = sm[warp] + x - v;
    *total = sm[kSampleWarps];
    __syncthreads();
    return r;
}

template <int STRATEGY>
__global__ void __launch_bounds__(kSampleThreads) sample_kernel(const __grid_constant__ SampleParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_scan[kSampleWarps + 1];
    __shared__ uint64_t s_base[TGL_MAX_SNAPSHOTS];
    __shared__ uint32_t s_tot[TGL_MAX_SNAPSHOTS];
    __shared__ uint32_t s_tile;

    constexpr int R = kSampleThreads;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nsb = p.nsb;
    const int k = p.k;

    uint32_t* incl = reinterpret_cast<uint32_t*>(smem);  // [nsb][R] counts -> inclusive prefix
    uint32_t* start = incl + nsb * R;                      // [nsb][R] first slot (most_recent) / a (uniform)
    float* troot = reinterpret_cast<float*>(start + nsb * R);  // [R]
    float* lo_r = troot + R;                                    // [nsb][R] window lower bound L
    uint64_t* rkey = reinterpret_cast<uint64_t*>(lo_r + nsb * R);  // [R] (offset is a multiple of 2R floats)

    if (tid == 0) s_tile = atomicAdd(p.tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;

    int64_t n = p.n_roots;
    if (p.n_roots_dev_in) {
        const int64_t m = *p.n_roots_dev_in;
        n = m < n ? m : n;
    }
    if (n <= 0) {
        if (tile == 0 && tid < nsb) {
            p.out[tid].offsets[0] = 0;
            *p.out[tid].nnz_dev = 0;
            *p.out[tid].n_roots_dev = 0;
        }
        return;
    }
    const int64_t base_i = (int64_t)tile * R;
    if (base_i >= n) return;  // capacity-sized grid: nobody waits on tiles past the end
    const int64_t i = base_i + tid;
    const bool valid = i < n;

    uint32_t* picks = nullptr;
    if (STRATEGY == TGL_UNIFORM)
        picks = p.picks_global ? p.picks_global + (size_t)tile * nsb * k * R
                               : reinterpret_cast<uint32_t*>(rkey + R);

    // ------------------------------------------------------------------ phase 1: cuts + selection
    int32_t v = 0;
    float t = 0.0f;
    bool ok = false;
    if (valid) {
        v = p.root_node[i];
        t = p.root_ts[i];
        if ((uint32_t)v >= (uint32_t)p.n_nodes)
            atomicOr(p.err, kErrRange);
        else if (!isfinite(t))
            atomicOr(p.err, kErrInval);
        else
            ok = true;
    }
    troot[tid] = t;
    uint64_t rk = 0;
    if (STRATEGY == TGL_UNIFORM) {
        rk = p.layer == 0 ? p.root_key_base + (uint64_t)i : (valid ? p.root_key[i] : 0ull);
        rkey[tid] = rk;
    }
    float lin = -INFINITY;
    if (p.layer > 0 && p.root_lo && ok) lin = p.root_lo[i];

    uint32_t lo = 0, hi = 0;
    if (ok) {
        lo = (uint32_t)__ldg(p.indptr + v);
        hi = (uint32_t)__ldg(p.indptr + v + 1);
    }
    // U of window 0 is the root's own time t (both for layer 0 and for hop roots)
    uint32_t bcur = ok ? lower_bound_ts(p.ts, lo, hi, t) : lo;
    for (int b = 0; b < nsb; ++b) {
        // lower bound of window b: layer 0 -> t (-) ((b+1) (x) t_s); l >= 1 -> inherited
        const float x = p.layer == 0 ? __fsub_rn(t, __fmul_rn((float)(b + 1), p.snapshot_len)) : lin;
        const uint32_t a = (ok && x > -INFINITY) ? lower_bound_ts(p.ts, lo, bcur, x) : lo;
        const uint32_t c = ok ? bcur - a : 0u;
        const uint32_t take = c < (uint32_t)k ? c : (uint32_t)k;
        incl[b * R + tid] = take;
        lo_r[b * R + tid] = x;
        if (STRATEGY == TGL_MOST_RECENT) {
            start[b * R + tid] = bcur - take;
        } else {
            start[b * R + tid] = a;
            uint32_t* pk = picks + (size_t)b * k * R + tid;  // pick q at pk[q * R]
            if (c <= (uint32_t)k) {
                for (uint32_t q = 0; q < c; ++q) pk[q * R] = q;
            } else {
                // Floyd: for m = c-k .. c-1, r uniform in [0, m]; take r unless taken, else m
                const uint32_t ctr1 = ((uint32_t)p.layer << 16) | (uint32_t)(p.layer == 0 ? b : p.snap0);
                for (int j = 0; j < k; ++j) {
                    const uint32_t m = c - (uint32_t)k + (uint32_t)j;
                    const uint4 rnd = philox4x32_10(make_uint4((uint32_t)j, ctr1, (uint32_t)rk, (uint32_t)(rk >> 32)),
                                                    p.seed_lo, p.seed_hi);
                    const uint32_t r = __umulhi(rnd.x, m + 1u);
                    bool taken = false;
                    for (int q = 0; q < j; ++q) taken |= (pk[q * R] == r);
                    pk[j * R] = taken ? m : r;
                }
                for (int j = 1; j < k; ++j) {  // ascending slot order (R#13)
                    const uint32_t xj = pk[j * R];
                    int q = j - 1;
                    while (q >= 0 && pk[q * R] > xj) {
                        pk[(q + 1) * R] = pk[q * R];
                        --q;
                    }
                    pk[(q + 1) * R] = xj;
                }
            }
        }
        bcur = a;
    }
    __syncthreads();

    // ------------------------------------------------------------------ phase 2: offsets
    for (int b = 0; b < nsb; ++b) {
        const uint32_t c = incl[b * R + tid];
        uint32_t tot;
        const uint32_t ex = block_excl_scan(c, &tot, s_scan);
        incl[b * R + tid] = ex + c;
        if (tid == 0) s_tot[b] = tot;
    }
    __syncthreads();
    for (int b = warp; b < nsb; b += kSampleWarps) {
        uint64_t* st = p.tile_state + (size_t)b * p.tiles_cap;
        const uint64_t agg = s_tot[b];
        if (lane == 0) st_relaxed_u64(st + tile, (tile == 0 ? kFlagPrefix : kFlagAgg) | agg);
        uint64_t excl = 0;
        if (tile > 0) {
            int64_t pred = (int64_t)tile - 1;
            while (true) {
                const int64_t idx = pred - lane;
                uint64_t w = idx >= 0 ? ld_relaxed_u64(st + idx) : kFlagPrefix;
                while (__any_sync(kFull, (w >> 62) == 0)) {
                    if ((w >> 62) == 0) w = ld_relaxed_u64(st + idx);
                }
                const uint32_t pm = __ballot_sync(kFull, (w >> 62) == 2);
                uint64_t val = w & kValMask;
                if (pm) {
                    const int first = __ffs(pm) - 1;
                    if (lane > first) val = 0;
                    excl += warp_sum_u64(val);
                    break;
                }
                excl += warp_sum_u64(val);
                pred -= 32;
            }
            if (lane == 0) st_relaxed_u64(st + tile, kFlagPrefix | (excl + agg));
        }
        if (lane == 0) s_base[b] = excl;
    }
    __syncthreads();

    const bool last_tile = base_i + R >= n;
    for (int b = 0; b < nsb; ++b) {
        const BlockOut& o = p.out[b];
        const uint32_t inc = incl[b * R + tid];
        const uint32_t ex = tid ? incl[b * R + tid - 1] : 0u;
        if (valid) o.offsets[i] = (int64_t)(s_base[b] + ex);
        if (last_tile && i == n - 1) {
            const int64_t total = (int64_t)(s_base[b] + inc);
            o.offsets[n] = total;
            *o.nnz_dev = total;
            *o.n_roots_dev = n;
        }
    }

    // ------------------------------------------------------------------ phase 3: flat copy
    for (int b = 0; b < nsb; ++b) {
        const BlockOut& o = p.out[b];
        const uint32_t T = s_tot[b];
        const uint64_t B = s_base[b];
        const uint32_t* inc = incl + b * R;
        const uint32_t* stb = start + b * R;
        for (uint32_t o0 = 0; o0 < T; o0 += R * kCopyUnroll) {
            uint32_t pos[kCopyUnroll], rr[kCopyUnroll], qq[kCopyUnroll];
            bool act[kCopyUnroll];
#pragma unroll
            for (int u = 0; u < kCopyUnroll; ++u) {
                const uint32_t oi = o0 + (uint32_t)(u * R + tid);
                act[u] = oi < T;
                // root of output oi: first r with inc[r] > oi
                uint32_t lo2 = 0, hi2 = R;
                while (lo2 < hi2) {
                    const uint32_t mid = (lo2 + hi2) >> 1;
                    if (inc[mid] <= oi)
                        lo2 = mid + 1;
                    else
                        hi2 = mid;
                }
                const uint32_t r = act[u] ? lo2 : 0u;
                const uint32_t q = act[u] ? oi - (r ? inc[r - 1] : 0u) : 0u;
                rr[u] = r;
                qq[u] = q;
                if (STRATEGY == TGL_MOST_RECENT)
                    pos[u] = stb[r] + q;
                else
                    pos[u] = act[u] ? stb[r] + picks[((size_t)b * k + q) * R + r] : 0u;
            }
            int32_t nb[kCopyUnroll], ed[kCopyUnroll];
            float tv[kCopyUnroll];
#pragma unroll
            for (int u = 0; u < kCopyUnroll; ++u) {
                if (act[u]) {
                    nb[u] = __ldg(p.nbr + pos[u]);
                    ed[u] = __ldg(p.eid + pos[u]);
                    tv[u] = __ldg(p.ts + pos[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < kCopyUnroll; ++u) {
                if (!act[u]) continue;
                const uint64_t oi = B + o0 + (uint32_t)(u * R + tid);
                o.nbr[oi] = nb[u];
                o.eid[oi] = ed[u];
                o.dt[oi] = __fsub_rn(troot[rr[u]], tv[u]);
                if (o.ts_edge) o.ts_edge[oi] = tv[u];
                if (o.child_key) o.child_key[oi] = rkey[rr[u]] * (uint64_t)k + qq[u];
                if (o.child_lo) o.child_lo[oi] = lo_r[b * R + rr[u]];
            }
        }
    }
}

static size_t sample_smem_bytes(int nsb, int k, int strategy, bool picks_in_smem) {
    const size_t R = kSampleThreads;
    size_t b = (size_t)nsb * R * 4 * 3 + R * 4;  // incl, start, lo_r, troot
    b += R * 8;                                  // rkey
    if (strategy == TGL_UNIFORM && picks_in_smem) b += (size_t)nsb * k * R * 4;
    return b;
}

static bool picks_fit_smem(int nsb, int k) { return (size_t)nsb * k * kSampleThreads * 4 <= kPicksSmemLimit; }

struct Launch {
    int layer, chain, nsb;
    int64_t roots_cap, tiles_cap;
    uint32_t* counter;
    uint64_t* state;
    uint32_t* picks;  // global picks or null
};

struct SamplePlan {
    int L = 0, S = 0;
    int64_t roots_cap[64], edges_cap[64];
    Launch launches[1 + 63 * TGL_MAX_SNAPSHOTS];
    int n_launch = 0;
    size_t memset_bytes = 0;
    uint64_t* child_key[64][TGL_MAX_SNAPSHOTS];
    float* child_lo[64][TGL_MAX_SNAPSHOTS];
    size_t bytes = 0;
};

static int plan_sample(int64_t n_roots, int L, const int32_t* fanouts, int S, int strategy, float snapshot_len,
                       void* ws, SamplePlan& P) {
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
    // tile counters + look-back state first: one contiguous region, one memset per call
    P.n_launch = 0;
    auto add = [&](int layer, int chain, int nsb) {
        Launch& la = P.launches[P.n_launch++];
        la.layer = layer;
        la.chain = chain;
        la.nsb = nsb;
        la.roots_cap = P.roots_cap[layer];
        la.tiles_cap = std::max<int64_t>(1, (la.roots_cap + kSampleThreads - 1) / kSampleThreads);
    };
    add(0, 0, S);
    for (int l = 1; l < L; ++l)
        for (int s = 0; s < S; ++s) add(l, s, 1);
    for (int j = 0; j < P.n_launch; ++j) {
        Launch& la = P.launches[j];
        la.counter = c.take<uint32_t>(64);
        la.state = c.take<uint64_t>((size_t)la.nsb * la.tiles_cap);
    }
    P.memset_bytes = c.bytes();
    const bool need_lo = L > 1 && std::isfinite(snapshot_len);
    for (int l = 0; l < L - 1; ++l)
        for (int s = 0; s < S; ++s) {
            P.child_key[l][s] = strategy == TGL_UNIFORM ? c.take<uint64_t>((size_t)P.edges_cap[l]) : nullptr;
            P.child_lo[l][s] = need_lo ? c.take<float>((size_t)P.edges_cap[l]) : nullptr;
        }
    for (int j = 0; j < P.n_launch; ++j) {
        Launch& la = P.launches[j];
        const int k = fanouts[la.layer];
        la.picks = nullptr;
        if (strategy == TGL_UNIFORM && !picks_fit_smem(la.nsb, k))
            la.picks = c.take<uint32_t>((size_t)la.tiles_cap * la.nsb * k * kSampleThreads);
    }
    P.bytes = c.bytes();
    return TGL_OK;
}

}  // namespace tgl

using namespace tgl;

extern "C" int tgl_sample_capacity(int64_t n_roots, int32_t n_layers, const int32_t* fanouts, int32_t n_snapshots,
                                   tgl_strategy strategy, float snapshot_len, int64_t* roots_cap, int64_t* edges_cap,
                                   size_t* ws_bytes) {
    static thread_local SamplePlan P;
    int rc = plan_sample(n_roots, n_layers, fanouts, n_snapshots, (int)strategy, snapshot_len, nullptr, P);
    if (rc) return rc;
    for (int l = 0; l < n_layers; ++l) {
        if (roots_cap) roots_cap[l] = P.roots_cap[l];
        if (edges_cap) edges_cap[l] = P.edges_cap[l];
    }
    if (ws_bytes) *ws_bytes = P.bytes;
    return TGL_OK;
}

extern "C" int tgl_sample(const tgl_tcsr* g, const int32_t* roots, const float* root_ts, int64_t n_roots,
                          int32_t n_layers, const int32_t* fanouts, tgl_strategy strategy, int32_t n_snapshots,
                          float snapshot_len, uint64_t seed, uint64_t root_key_base, tgl_block* out, void* workspace,
                          size_t ws_bytes, void* stream) {
    if (!g || !out || !workspace) return TGL_EINVAL;
    if (n_roots > 0 && (!roots || !root_ts)) return TGL_EINVAL;
    static thread_local SamplePlan P;
    int rc = plan_sample(n_roots, n_layers, fanouts, n_snapshots, (int)strategy, snapshot_len, workspace, P);
    if (rc) return rc;
    if (ws_bytes < P.bytes) return TGL_EWORKSPACE;
    rc = check_device();
    if (rc) return rc;
    const int L = n_layers, S = n_snapshots;
    for (int l = 0; l < L; ++l)
        for (int s = 0; s < S; ++s) {
            const tgl_block& b = out[l * S + s];
            if (!b.offsets || !b.nbr || !b.eid || !b.dt || !b.n_roots_dev || !b.nnz_dev) return TGL_EINVAL;
            if (l < L - 1 && !b.ts_edge) return TGL_EINVAL;
            if (b.cap_roots < P.roots_cap[l] || b.cap_edges < P.edges_cap[l]) return TGL_ECAPACITY;
        }
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(workspace, 0, P.memset_bytes, st) != cudaSuccess) return TGL_ECUDA;

    for (int j = 0; j < P.n_launch; ++j) {
        const Launch& la = P.launches[j];
        const int l = la.layer, s = la.chain;
        SampleParams sp;
        memset(&sp, 0, sizeof(sp));
        sp.indptr = g->indptr;
        sp.nbr = g->nbr;
        sp.ts = g->ts;
        sp.eid = g->eid;
        sp.n_nodes = g->n_nodes;
        if (l == 0) {
            sp.root_node = roots;
            sp.root_ts = root_ts;
            sp.root_key = nullptr;
            sp.root_lo = nullptr;
            sp.n_roots = n_roots;
            sp.n_roots_dev_in = nullptr;
        } else {
            const tgl_block& par = out[(l - 1) * S + s];
            sp.root_node = par.nbr;
            sp.root_ts = par.ts_edge;
            sp.root_key = P.child_key[l - 1][s];
            sp.root_lo = P.child_lo[l - 1][s];
            sp.n_roots = P.roots_cap[l];
            sp.n_roots_dev_in = par.nnz_dev;
        }
        sp.root_key_base = root_key_base;
        sp.layer = l;
        sp.nsb = la.nsb;
        sp.snap0 = s;
        sp.k = fanouts[l];
        sp.snapshot_len = snapshot_len;
        sp.seed_lo = (uint32_t)seed;
        sp.seed_hi = (uint32_t)(seed >> 32);
        sp.tile_state = la.state;
        sp.tile_counter = la.counter;
        sp.tiles_cap = la.tiles_cap;
        sp.picks_global = la.picks;
        sp.err = g->err_dev;
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
            bo.n_roots_dev = ob.n_roots_dev;
            bo.nnz_dev = ob.nnz_dev;
        }
        const int64_t grid = l == 0 ? std::max<int64_t>(1, (n_roots + kSampleThreads - 1) / kSampleThreads)
                                    : la.tiles_cap;
        const bool in_smem = la.picks == nullptr;
        const size_t smem = sample_smem_bytes(la.nsb, sp.k, (int)strategy, in_smem);
        if (strategy == TGL_UNIFORM) {
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(sample_kernel<TGL_UNIFORM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
            sample_kernel<TGL_UNIFORM><<<(unsigned)grid, kSampleThreads, smem, st>>>(sp);
        } else {
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(sample_kernel<TGL_MOST_RECENT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
            sample_kernel<TGL_MOST_RECENT><<<(unsigned)grid, kSampleThreads, smem, st>>>(sp);
        }
        if (cudaGetLastError() != cudaSuccess) return TGL_ECUDA;
    }
    return TGL_OK;
}
