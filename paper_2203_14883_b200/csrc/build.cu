// build.cu -- T-CSR construction on B200 (Sec. 3.1 "The T-CSR Data Structure").
//
//   K1 validate_hist_kernel   a1 + a2: range / finiteness / chronology checks (device flags) and
//                             the owner-degree histogram (warp-aggregated atomics).
//   K2 exclusive_scan         a3: indptr[v] = sum_{u<v} deg[u], indptr[V] = E_s.
//   K3 radix passes           a4: the stable scatter.  The slot of logical edge j is
//                             indptr[owner_j] + #{j' < j : owner_j' = owner_j}.  Computed as a
//                             stable LSD counting sort of (owner, j) by owner, 8 bits per pass:
//                             each pass is itself histogram -> scan -> stable scatter, with the
//                             in-tile stable rank from __match_any_sync.  The last pass writes
//                             the T-CSR arrays directly at the final slot (the sort position IS
//                             the slot), so lists come out in stream = time order without a
//                             sort on time, ties by stream order (R#8).
//
// Deterministic: no atomic decides an output position.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "radix.cuh"
#include "scan.cuh"
#include "tsindex.cuh"

namespace tgl {


// ---------------------------------------------------------------------------- K1
__global__ void __launch_bounds__(256) validate_hist_kernel(const int32_t* __restrict__ src,
                                                            const int32_t* __restrict__ dst,
                                                            const float* __restrict__ ts, int64_t n,
                                                            int32_t n_nodes, int add_reverse, int32_t node_lo,
                                                            int32_t node_hi, uint32_t* __restrict__ deg,
                                                            int* __restrict__ err) {
    int bits = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i - threadIdx.x % 32 < n; i += stride) {
        const bool live = i < n;
        int32_t s = 0, d = 0;
        if (live) {
            s = src[i];
            d = dst[i];
            const float t = ts[i];
            if (!(t >= 0.0f && t <= 3.402823466e38f)) bits |= kErrInval;  // NaN, inf, negative
            if (i > 0 && ts[i - 1] > t) bits |= kErrUnsorted;
            if ((uint32_t)s >= (uint32_t)n_nodes || (uint32_t)d >= (uint32_t)n_nodes) bits |= kErrRange;
        }
        // owners counted: those in [node_lo, node_hi) (the whole graph, or one node-sharded range)
        const bool ok_s = live && s >= node_lo && s < node_hi;
        const bool ok_d = live && add_reverse && d >= node_lo && d < node_hi;
        // warp-aggregated histogram: one atomic per distinct owner in the warp
        {
            const int key = ok_s ? s : -1;
            const uint32_t peers = __match_any_sync(kFull, key);
            if (ok_s && (__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&deg[s - node_lo], __popc(peers));
        }
        if (add_reverse) {
            const int key = ok_d ? d : -1;
            const uint32_t peers = __match_any_sync(kFull, key);
            if (ok_d && (__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&deg[d - node_lo], __popc(peers));
        }
    }
    bits = __reduce_or_sync(kFull, bits);
    if (bits && (threadIdx.x & 31) == 0) atomicOr(err, bits);
}

// ---------------------------------------------------------------------------- host plan
struct BuildPlan {
    uint64_t n_logical = 0;
    int bits = 0, passes = 1;
    uint64_t ntiles = 0;
    int nbuf = 0;
    int* err = nullptr;
    uint32_t* deg = nullptr;
    uint64_t* partial = nullptr;
    uint32_t* counts = nullptr;
    uint32_t* kbuf[2] = {nullptr, nullptr};
    uint32_t* vbuf[2] = {nullptr, nullptr};
    size_t bytes = 0;
};

static BuildPlan plan_build(int64_t n_edges, int32_t n_nodes, int add_reverse, void* ws) {
    BuildPlan p;
    p.n_logical = (uint64_t)n_edges * (add_reverse ? 2 : 1);
    p.bits = n_nodes <= 1 ? 0 : 32 - __builtin_clz((unsigned)(n_nodes - 1));
    p.passes = p.bits <= 8 ? 1 : (p.bits + 7) / 8;
    p.ntiles = (p.n_logical + kRadixTile - 1) / kRadixTile;
    p.nbuf = p.passes >= 3 ? 2 : (p.passes == 2 ? 1 : 0);
    Carve c(ws);
    p.err = c.take<int>(64);
    p.deg = c.take<uint32_t>((size_t)(n_nodes > 0 ? n_nodes : 1));
    int64_t scan_n = std::max<int64_t>((int64_t)n_nodes, (int64_t)(kRadixBins * p.ntiles));
    p.partial = c.take<uint64_t>(scan_workspace_bytes(scan_n) / sizeof(uint64_t));
    p.counts = c.take<uint32_t>((size_t)kRadixBins * (p.ntiles ? p.ntiles : 1));
    for (int b = 0; b < p.nbuf; ++b) {
        p.kbuf[b] = c.take<uint32_t>(p.n_logical);
        p.vbuf[b] = c.take<uint32_t>(p.n_logical);
    }
    p.bytes = c.bytes();
    return p;
}

}  // namespace tgl

using namespace tgl;

extern "C" int tgl_tcsr_build_workspace(int64_t n_edges, int32_t n_nodes, int add_reverse, size_t* bytes) {
    if (!bytes || n_edges < 0 || n_nodes < 0) return TGL_EINVAL;
    const uint64_t es = (uint64_t)n_edges * (add_reverse ? 2 : 1);
    if (es >= (1ull << 32)) return TGL_EINVAL;
    *bytes = plan_build(n_edges, n_nodes, add_reverse ? 1 : 0, nullptr).bytes;
    return TGL_OK;
}

namespace tgl {
// ---------------------------------------------------------------------------- aux: time codec
// (tsindex.cuh "time codes").  X1 collects the distinct timestamp bits (at most kMaxCodes; any
// negative, -0, infinite or NaN time disables the codec): warp leaders of equal values
// (__match_any_sync) insert into a per-CTA hash in shared memory, merged into a global hash at
// the end.  X2 (one CTA) ranks them -- non-negative finite floats order like their bit patterns
// -- into the sorted dictionary.  X3 writes every slot's code and the per-code eid range and the
// largest neighbour id (the packed record widths).
__device__ __forceinline__ uint32_t hash_bits(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    return x;
}

__global__ void __launch_bounds__(256) codec_collect_kernel(const float* __restrict__ ts, uint64_t n,
                                                            CodecScratch* sc) {
    __shared__ uint32_t h[512];
    __shared__ uint32_t cnt;
    for (int q = threadIdx.x; q < 512; q += blockDim.x) h[q] = 0xffffffffu;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    bool ovf = false;  // block-uniform (__syncthreads_or)
    for (uint64_t j0 = (uint64_t)blockIdx.x * blockDim.x; j0 < n && !ovf; j0 += stride) {
        const uint64_t j = j0 + threadIdx.x;
        const bool live = j < n;
        const uint32_t bits = live ? __float_as_uint(ts[j]) : 0xffffffffu;
        bool bad = live && bits >= 0x7f800000u;  // +inf, NaN, or sign bit set (negative, -0)
        const uint32_t peers = __match_any_sync(kFull, bits);
        if (live && !bad && (__ffs(peers) - 1) == (int)(threadIdx.x & 31)) {
            uint32_t slot = hash_bits(bits) & 511u;
            bool done = false;
            for (int probe = 0; probe < 512 && !done; ++probe) {
                const uint32_t prev = atomicCAS(&h[slot], 0xffffffffu, bits);
                if (prev == 0xffffffffu) {
                    bad |= atomicAdd(&cnt, 1u) >= (uint32_t)kMaxCodes;
                    done = true;
                } else if (prev == bits) {
                    done = true;
                }
                slot = (slot + 1) & 511u;
            }
            bad |= !done;
        }
        if (threadIdx.x == 0) bad |= *reinterpret_cast<volatile uint32_t*>(&sc->overflow) != 0u;
        ovf = __syncthreads_or(bad) != 0;
    }
    if (ovf) {
        if (threadIdx.x == 0) atomicOr(&sc->overflow, 1u);
        return;
    }
    for (int q = threadIdx.x; q < 512; q += blockDim.x) {
        const uint32_t bits = h[q];
        if (bits == 0xffffffffu) continue;
        uint32_t slot = hash_bits(bits) & 511u;
        bool done = false;
        for (int probe = 0; probe < 512 && !done; ++probe) {
            const uint32_t prev = atomicCAS(&sc->hash[slot], 0xffffffffu, bits);
            if (prev == 0xffffffffu) {
                if (atomicAdd(&sc->count, 1u) >= (uint32_t)kMaxCodes) atomicOr(&sc->overflow, 1u);
                done = true;
            } else if (prev == bits) {
                done = true;
            }
            slot = (slot + 1) & 511u;
        }
        if (!done) atomicOr(&sc->overflow, 1u);
    }
}

__global__ void __launch_bounds__(512) codec_dict_kernel(CodecScratch* sc, TimeDict* dict) {
    __shared__ uint32_t h[512];
    const int q = threadIdx.x;
    h[q] = sc->hash[q];
    if (q < 256) {
        dict->value[q] = INFINITY;
        dict->eid_base[q] = 0;
        sc->eid_min[q] = INT32_MAX;
        sc->eid_max[q] = INT32_MIN;
    }
    __syncthreads();
    const uint32_t b = h[q];
    if (b != 0xffffffffu) {
        uint32_t rank = 0;
        for (int r = 0; r < 512; ++r) rank += h[r] != 0xffffffffu && h[r] < b;
        dict->value[rank] = __uint_as_float(b);
    }
}

__global__ void __launch_bounds__(256) codec_assign_kernel(const float* __restrict__ ts, const int32_t* __restrict__ nbr,
                                                           const int32_t* __restrict__ eid, uint64_t n,
                                                           const TimeDict* __restrict__ dict,
                                                           uint8_t* __restrict__ codes, CodecScratch* sc) {
    __shared__ float val[256];
    __shared__ int32_t emin[256], emax[256];
    __shared__ uint32_t nmax;
    val[threadIdx.x] = dict->value[threadIdx.x];
    emin[threadIdx.x] = INT32_MAX;
    emax[threadIdx.x] = INT32_MIN;
    if (threadIdx.x == 0) nmax = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t my_nmax = 0;
    for (uint64_t j0 = (uint64_t)blockIdx.x * blockDim.x; j0 < n; j0 += stride) {
        const uint64_t j = j0 + threadIdx.x;
        const bool live = j < n;
        uint32_t c = 0xffffffffu;
        int32_t e = 0;
        if (live) {
            const float t = ts[j];
            uint32_t lo = 0;  // #values < t = the index of t (t is in the dictionary)
#pragma unroll
            for (int step = 128; step >= 1; step >>= 1)
                if (val[lo + step - 1] < t) lo += step;
            c = lo;
            codes[j] = (uint8_t)c;
            e = eid[j];
            my_nmax = max(my_nmax, (uint32_t)nbr[j]);
        }
        const uint32_t peers = __match_any_sync(kFull, c);
        const int32_t mn = __reduce_min_sync(peers, live ? e : INT32_MAX);
        const int32_t mx = __reduce_max_sync(peers, live ? e : INT32_MIN);
        if (live && (__ffs(peers) - 1) == (int)(threadIdx.x & 31)) {
            atomicMin(&emin[c], mn);
            atomicMax(&emax[c], mx);
        }
    }
    my_nmax = __reduce_max_sync(kFull, my_nmax);
    if ((threadIdx.x & 31) == 0) atomicMax(&nmax, my_nmax);
    __syncthreads();
    if (emin[threadIdx.x] != INT32_MAX) {
        atomicMin(&sc->eid_min[threadIdx.x], emin[threadIdx.x]);
        atomicMax(&sc->eid_max[threadIdx.x], emax[threadIdx.x]);
    }
    if (threadIdx.x == 0) atomicMax(&sc->nbr_max, nmax);
}

// integer-time packing (packed = 2, tsindex.cuh): are all times integers in [0, 2^24), their
// largest value, the eid range and the largest neighbour id
__global__ void __launch_bounds__(256) inttime_scan_kernel(const float* __restrict__ ts, const int32_t* __restrict__ nbr,
                                                           const int32_t* __restrict__ eid, uint64_t n,
                                                           CodecScratch* sc) {
    uint32_t tmax = 0, bad = 0, nmax = 0;
    int32_t emn = INT32_MAX, emx = INT32_MIN;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        const float t = ts[j];
        const uint32_t bits = __float_as_uint(t);
        // integers in [0, 2^24): sign clear, below 2^24, no fraction
        bad |= (bits >= 0x4b800000u || t != truncf(t)) ? 1u : 0u;
        tmax = max(tmax, bits);
        nmax = max(nmax, (uint32_t)nbr[j]);
        emn = min(emn, eid[j]);
        emx = max(emx, eid[j]);
    }
    tmax = __reduce_max_sync(kFull, tmax);
    bad = __reduce_or_sync(kFull, bad);
    nmax = __reduce_max_sync(kFull, nmax);
    emn = __reduce_min_sync(kFull, emn);
    emx = __reduce_max_sync(kFull, emx);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&sc->t_max_bits, tmax);
        atomicOr(&sc->not_int, bad);
        atomicMax(&sc->nbr_max, nmax);
        atomicMin(&sc->e_min, emn);
        atomicMax(&sc->e_max, emx);
    }
}

struct CodecArgs {
    const uint8_t* codes;   // null: no codec
    const int32_t* eid_base;
    int packed, bn, bc;  // packed: 1 time codes, 2 integer times (bc = eid offset width)
    int32_t ebase0;      // packed = 2: the smallest eid
};

// aux buffer (tsindex.cuh): index levels L_l[j] = ts[j * 16^l], the slot records (16-byte, or
// 8-byte packed) and the node records (14 fence times, or 54 fence codes under the time codec)
__global__ void aux_build_kernel(const int64_t* __restrict__ indptr, const float* __restrict__ ts,
                                 const int32_t* __restrict__ nbr, const int32_t* __restrict__ eid, uint64_t n,
                                 uint64_t n_nodes, char* __restrict__ aux, AuxLayout lay, CodecArgs cx) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    float* index = reinterpret_cast<float*>(aux + lay.index_off);
    for (int l = 1; l <= lay.index.n_levels; ++l) {
        float* out = index + lay.index.off[l];
        const int sh = kIndexShift * l;
        for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < lay.index.len[l]; j += stride)
            out[j] = ts[j << sh];
    }
    if (cx.packed == 1) {
        uint2* rec = reinterpret_cast<uint2*>(aux + lay.rec_off);
        for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
            const uint32_t c = cx.codes[j];
            const uint64_t rel = (uint64_t)(uint32_t)(eid[j] - __ldg(cx.eid_base + c));
            const uint64_t w = (uint64_t)(uint32_t)nbr[j] | ((uint64_t)c << cx.bn) | (rel << (cx.bn + cx.bc));
            rec[j] = make_uint2((uint32_t)w, (uint32_t)(w >> 32));
        }
    } else if (cx.packed == 2) {
        uint2* rec = reinterpret_cast<uint2*>(aux + lay.rec_off);
        for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
            const uint64_t rel = (uint64_t)(uint32_t)(eid[j] - cx.ebase0);
            const uint64_t tint = (uint64_t)(uint32_t)ts[j];
            const uint64_t w = (uint64_t)(uint32_t)nbr[j] | (rel << cx.bn) | (tint << (cx.bn + cx.bc));
            rec[j] = make_uint2((uint32_t)w, (uint32_t)(w >> 32));
        }
    } else {
        SlotRec* rec = reinterpret_cast<SlotRec*>(aux + lay.rec_off);
        for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
            SlotRec r;
            memset(&r, 0, sizeof(r));
            r.ts = ts[j];
            r.nbr = nbr[j];
            r.eid = eid[j];
            rec[j] = r;
        }
    }
    // node records: thread (v, q) writes the q-th 16-byte quarter of node v's record
    int4* node = reinterpret_cast<int4*>(aux + lay.node_off);
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n_nodes * 4; w += stride) {
        const uint64_t v = w >> 2;
        const int q = (int)(w & 3);
        const uint32_t lo = (uint32_t)indptr[v], hi = (uint32_t)indptr[v + 1], d = hi - lo;
        int32_t word[4];
        if (cx.codes) {  // {lo, hi, 10 separators + 2 pads, 11 groups of 4} (tsindex.cuh)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int wi = 4 * q + e;  // record word
                if (wi < 2) {
                    word[e] = (int32_t)(wi == 0 ? lo : hi);
                    continue;
                }
                uint32_t x = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    int j;  // fence index of byte b of word wi (-1: pad)
                    if (wi < 5) {
                        const int sep = 4 * (wi - 2) + b;
                        j = sep < kCodeSeps ? 5 * sep + 4 : -1;
                    } else {
                        j = 5 * (wi - 5) + b;
                    }
                    const uint32_t c = (j < 0 || d == 0) ? kCodeInf : cx.codes[code_fence_pos(lo, d, j)];
                    x |= c << (8 * b);
                }
                word[e] = (int32_t)x;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = 4 * q + e - 2;  // fence index of word e (words 0, 1 of quarter 0: lo, hi)
                word[e] = j < 0 ? (int32_t)(j == -2 ? lo : hi)
                                : __float_as_int(d ? ts[fence_pos(lo, d, j)] : INFINITY);
            }
        }
        node[w] = make_int4(word[0], word[1], word[2], word[3]);
    }
}

static int bit_width(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

}  // namespace tgl

extern "C" int tgl_tcsr_aux_bytes(int64_t n_stored, int32_t n_nodes, size_t* bytes) {
    if (!bytes || n_stored < 0 || n_nodes < 0 || (uint64_t)n_stored >= (1ull << 32)) return TGL_EINVAL;
    *bytes = aux_layout((uint64_t)n_stored, (uint64_t)n_nodes).bytes;
    return TGL_OK;
}

extern "C" int tgl_tcsr_aux_build(const int64_t* indptr, const float* ts, const int32_t* nbr, const int32_t* eid,
                                  int32_t n_nodes, int64_t n_stored, void* aux, size_t aux_bytes, void* stream) {
    if (n_stored < 0 || n_nodes < 0 || (uint64_t)n_stored >= (1ull << 32) || !aux || !indptr) return TGL_EINVAL;
    if (n_stored > 0 && (!ts || !nbr || !eid)) return TGL_EINVAL;
    const AuxLayout lay = aux_layout((uint64_t)n_stored, (uint64_t)n_nodes);
    if (aux_bytes < lay.bytes) return TGL_EWORKSPACE;
    int rc = check_device();
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    char* ab = static_cast<char*>(aux);
    TimeDict* dict = reinterpret_cast<TimeDict*>(ab);
    CodecScratch* sc = reinterpret_cast<CodecScratch*>(ab + sizeof(TimeDict));
    uint8_t* codes = reinterpret_cast<uint8_t*>(ab + lay.code_off);
    const uint64_t n = (uint64_t)n_stored;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 8));
    // X1: distinct times (<= kMaxCodes)
    if (cudaMemsetAsync(sc->hash, 0xff, sizeof(sc->hash), st) != cudaSuccess ||
        cudaMemsetAsync(&sc->count, 0, 4 * sizeof(uint32_t), st) != cudaSuccess)
        return TGL_ECUDA;
    if (n > 0) codec_collect_kernel<<<grid, 256, 0, st>>>(ts, n, sc);
    uint32_t cnt[2] = {0, 0};
    if (cudaMemcpyAsync(cnt, &sc->count, sizeof(cnt), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return TGL_ECUDA;
    static const bool no_codec = getenv("TGL_NO_CODEC") != nullptr;  // A/B knob, read once
    const uint32_t D = (n > 0 && !cnt[1] && !no_codec) ? cnt[0] : 0u;
    uint32_t hdr[8] = {kDictMagic, D, 0, 0, 0, 0, 0, 0};
    CodecArgs cx = {nullptr, nullptr, 0, 0, 0, 0};
    if (D > 0) {
        // X2 dictionary, X3 codes + widths
        codec_dict_kernel<<<1, 512, 0, st>>>(sc, dict);
        if (cudaMemsetAsync(&sc->nbr_max, 0, sizeof(uint32_t), st) != cudaSuccess) return TGL_ECUDA;
        codec_assign_kernel<<<grid, 256, 0, st>>>(ts, nbr, eid, n, dict, codes, sc);
        int32_t emin[256], emax[256];
        uint32_t nmax = 0;
        if (cudaMemcpyAsync(emin, sc->eid_min, sizeof(emin), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaMemcpyAsync(emax, sc->eid_max, sizeof(emax), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaMemcpyAsync(&nmax, &sc->nbr_max, sizeof(nmax), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return TGL_ECUDA;
        uint64_t span = 0;
        for (uint32_t c = 0; c < D; ++c) span = std::max<uint64_t>(span, (uint64_t)((int64_t)emax[c] - (int64_t)emin[c]));
        const int bn = bit_width(nmax), bc = bit_width(D - 1), br = bit_width(span);
        const bool packed = bn + bc + br <= 64;
        hdr[2] = packed ? 1u : 0u;
        hdr[3] = (uint32_t)bn;
        hdr[4] = (uint32_t)bc;
        if (cudaMemcpyAsync(dict->eid_base, emin, sizeof(emin), cudaMemcpyHostToDevice, st) != cudaSuccess)
            return TGL_ECUDA;
        cx = CodecArgs{codes, dict->eid_base, packed ? 1 : 0, bn, bc, 0};
    } else if (n > 0 && !no_codec) {
        // no time codes: integer times below 2^24 still pack (packed = 2, tsindex.cuh)
        const uint32_t init[6] = {0u, 0u, 0u, 0u, (uint32_t)INT32_MAX, (uint32_t)INT32_MIN};  // t_max, not_int, e_min, e_max
        if (cudaMemsetAsync(&sc->nbr_max, 0, sizeof(uint32_t), st) != cudaSuccess ||
            cudaMemcpyAsync(&sc->t_max_bits, init, 2 * sizeof(uint32_t), cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaMemcpyAsync(&sc->e_min, init + 4, 2 * sizeof(uint32_t), cudaMemcpyHostToDevice, st) != cudaSuccess)
            return TGL_ECUDA;
        inttime_scan_kernel<<<grid, 256, 0, st>>>(ts, nbr, eid, n, sc);
        uint32_t r[2] = {0, 0}, nmax = 0;
        int32_t e[2] = {0, 0};
        if (cudaMemcpyAsync(r, &sc->t_max_bits, sizeof(r), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaMemcpyAsync(e, &sc->e_min, sizeof(e), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaMemcpyAsync(&nmax, &sc->nbr_max, sizeof(nmax), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return TGL_ECUDA;
        float tmax = 0.0f;
        memcpy(&tmax, &r[0], sizeof(tmax));
        const int bn = bit_width(nmax), be = bit_width((uint64_t)((int64_t)e[1] - (int64_t)e[0])),
                  bt = bit_width((uint64_t)tmax);
        if (!r[1] && bn + be + bt <= 64) {
            hdr[2] = 2u;
            hdr[3] = (uint32_t)bn;
            hdr[4] = (uint32_t)be;
            hdr[5] = (uint32_t)e[0];
            cx = CodecArgs{nullptr, nullptr, 2, bn, be, e[0]};
        }
    }
    if (cudaMemcpyAsync(dict, hdr, sizeof(hdr), cudaMemcpyHostToDevice, st) != cudaSuccess) return TGL_ECUDA;
    const int64_t blocks = std::min<int64_t>((int64_t)((std::max<int64_t>(n_stored, (int64_t)n_nodes * 4) + 255) / 256),
                                             148 * 16);
    aux_build_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, st>>>(
        indptr, ts, nbr, eid, n, (uint64_t)n_nodes, ab, lay, cx);
    if (cudaGetLastError() != cudaSuccess) return TGL_ECUDA;
    // the host copies above read stack memory: complete them (and the buffer) before returning
    return cudaStreamSynchronize(st) == cudaSuccess ? TGL_OK : TGL_ECUDA;
}

extern "C" int tgl_tcsr_build(const int32_t* src, const int32_t* dst, const float* ts, const int32_t* eid,
                              int64_t n_edges, int32_t n_nodes, int add_reverse, int64_t* indptr, int32_t* nbr,
                              float* ts_out, int32_t* eid_out, void* aux, size_t aux_bytes, void* workspace,
                              size_t ws_bytes, void* stream, tgl_tcsr** out) {
    NvtxRange nvtx_("tgl_tcsr_build");
    if (!out || !indptr || n_edges < 0 || n_nodes < 0) return TGL_EINVAL;
    *out = nullptr;
    add_reverse = add_reverse ? 1 : 0;
    const uint64_t es = (uint64_t)n_edges * (add_reverse ? 2 : 1);
    if (es >= (1ull << 32)) return TGL_EINVAL;
    if (n_edges > 0 && (!src || !dst || !ts || !nbr || !ts_out || !eid_out)) return TGL_EINVAL;
    if (!workspace) return TGL_EINVAL;
    int rc = check_device();
    if (rc) return rc;
    BuildPlan p = plan_build(n_edges, n_nodes, add_reverse, workspace);
    if (ws_bytes < p.bytes) return TGL_EWORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;

    // K1: validation + degree histogram
    if (cudaMemsetAsync(p.err, 0, sizeof(int), st) != cudaSuccess) return TGL_ECUDA;
    if (n_nodes > 0 && cudaMemsetAsync(p.deg, 0, sizeof(uint32_t) * (size_t)n_nodes, st) != cudaSuccess)
        return TGL_ECUDA;
    if (n_edges > 0) {
        int64_t blocks = std::min<int64_t>((n_edges + 255) / 256, 148 * 16);
        validate_hist_kernel<<<(unsigned)blocks, 256, 0, st>>>(src, dst, ts, n_edges, n_nodes, add_reverse, 0,
                                                                n_nodes, p.deg, p.err);
        if (cudaGetLastError() != cudaSuccess) return TGL_ECUDA;
    }
    int herr = 0;
    if (cudaMemcpyAsync(&herr, p.err, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess) return TGL_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return TGL_ECUDA;
    if (herr) return err_bits_to_code(herr);

    // K2: indptr = exclusive scan of degrees, indptr[V] = E_s
    if (cuda_rc(exclusive_scan<uint32_t, int64_t>(p.deg, indptr, n_nodes, indptr + n_nodes, p.partial, st)))
        return TGL_ECUDA;

    // K3: stable scatter via LSD counting-sort passes over the logical stream
    if (p.n_logical > 0) {
        Stream s{src, dst, ts, eid, add_reverse};
        const uint64_t n = p.n_logical;
        for (int pass = 0; pass < p.passes; ++pass) {
            const int shift = 8 * pass;
            const int nb = std::min(8, std::max(0, p.bits - shift));
            const uint32_t mask = nb >= 32 ? 0xffffffffu : ((1u << nb) - 1u);
            const bool first = pass == 0, last = pass == p.passes - 1;
            const uint32_t* kin = first ? nullptr : p.kbuf[(pass - 1) & 1];
            const uint32_t* vin = first ? nullptr : p.vbuf[(pass - 1) & 1];
            uint32_t* kout = last ? nullptr : p.kbuf[pass & 1];
            uint32_t* vout = last ? nullptr : p.vbuf[pass & 1];
            const unsigned grid = (unsigned)p.ntiles;
            if (first)
                radix_upsweep_kernel<kSrcStream><<<grid, kRadixThreads, 0, st>>>(s, kin, n, shift, mask, p.counts,
                                                                                  p.ntiles);
            else
                radix_upsweep_kernel<kSrcKV><<<grid, kRadixThreads, 0, st>>>(s, kin, n, shift, mask, p.counts,
                                                                              p.ntiles);
            if (cuda_rc(exclusive_scan<uint32_t, uint32_t>(p.counts, p.counts, (int64_t)kRadixBins * p.ntiles,
                                                           (uint32_t*)nullptr, p.partial, st)))
                return TGL_ECUDA;
            if (first && last)
                radix_downsweep_kernel<kSrcStream, kDstTCSR><<<grid, kRadixThreads, 0, st>>>(
                    s, kin, vin, n, shift, mask, p.counts, p.ntiles, kout, vout, nbr, ts_out, eid_out, nullptr);
            else if (first)
                radix_downsweep_kernel<kSrcStream, kDstKV><<<grid, kRadixThreads, 0, st>>>(
                    s, kin, vin, n, shift, mask, p.counts, p.ntiles, kout, vout, nbr, ts_out, eid_out, nullptr);
            else if (last)
                radix_downsweep_kernel<kSrcKV, kDstTCSR><<<grid, kRadixThreads, 0, st>>>(
                    s, kin, vin, n, shift, mask, p.counts, p.ntiles, kout, vout, nbr, ts_out, eid_out, nullptr);
            else
                radix_downsweep_kernel<kSrcKV, kDstKV><<<grid, kRadixThreads, 0, st>>>(
                    s, kin, vin, n, shift, mask, p.counts, p.ntiles, kout, vout, nbr, ts_out, eid_out, nullptr);
            if (cudaGetLastError() != cudaSuccess) return TGL_ECUDA;
        }
    }
    if (aux) {
        rc = tgl_tcsr_aux_build(indptr, ts_out, nbr, eid_out, n_nodes, (int64_t)es, aux, aux_bytes, stream);
        if (rc) return rc;
    }
    return tgl_tcsr_wrap(indptr, nbr, ts_out, eid_out, aux, aux_bytes, n_nodes, (int64_t)es, out);
}

// ---------------------------------------------------------------------------- node-range build
// Node-sharded T-CSR: a rank builds only the lists of its node range [lo, hi), so its
// T-CSR memory is ~E_s / world.  Same method as tgl_tcsr_build, restricted to the
// logical edges whose owner is in the range: K1 (validation of the whole stream + the range's
// degree histogram), K2 (scan -> the local indptr), then the logical edges of the range are
// compacted in stream order (flag -> scan -> scatter of (owner - lo, j)) and sorted by the same
// stable LSD passes, so every list is exactly the full build's list of that node.
namespace tgl {

__global__ void range_flag_kernel(Stream s, uint64_t n, int32_t lo, int32_t hi, uint32_t* __restrict__ flag) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        const int32_t o = (int32_t)owner_of(s, j);
        flag[j] = o >= lo && o < hi ? 1u : 0u;
    }
}

__global__ void range_compact_kernel(Stream s, uint64_t n, int32_t lo, const uint32_t* __restrict__ flag,
                                     const uint32_t* __restrict__ pos, uint32_t* __restrict__ keys,
                                     uint32_t* __restrict__ vals) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
        if (flag[j]) {
            keys[pos[j]] = owner_of(s, j) - (uint32_t)lo;
            vals[pos[j]] = (uint32_t)j;
        }
}

struct RangePlan {
    uint64_t n_logical = 0, n_local = 0;
    int bits = 0, passes = 1;
    uint64_t ntiles = 0;
    int* err = nullptr;
    uint32_t* deg = nullptr;
    uint32_t* flag = nullptr;  // [n_logical], then reused as the compaction positions
    uint32_t* pos = nullptr;
    uint64_t* partial = nullptr;
    uint32_t* counts = nullptr;
    uint32_t* kbuf[2] = {nullptr, nullptr};
    uint32_t* vbuf[2] = {nullptr, nullptr};
    size_t bytes = 0;
};

static RangePlan plan_range(int64_t n_edges, int32_t n_local_nodes, int64_t n_local, int add_reverse, void* ws) {
    RangePlan p;
    p.n_logical = (uint64_t)n_edges * (add_reverse ? 2 : 1);
    p.n_local = (uint64_t)n_local;
    p.bits = n_local_nodes <= 1 ? 0 : 32 - __builtin_clz((unsigned)(n_local_nodes - 1));
    p.passes = p.bits <= 8 ? 1 : (p.bits + 7) / 8;
    p.ntiles = (p.n_local + kRadixTile - 1) / kRadixTile;
    Carve c(ws);
    p.err = c.take<int>(64);
    p.deg = c.take<uint32_t>((size_t)std::max(n_local_nodes, 1));
    p.flag = c.take<uint32_t>((size_t)std::max<uint64_t>(p.n_logical, 1));
    p.pos = c.take<uint32_t>((size_t)std::max<uint64_t>(p.n_logical, 1));
    const int64_t scan_n = std::max<int64_t>(std::max<int64_t>(n_local_nodes, (int64_t)p.n_logical),
                                             (int64_t)(kRadixBins * p.ntiles));
    p.partial = c.take<uint64_t>(scan_workspace_bytes(scan_n) / sizeof(uint64_t));
    p.counts = c.take<uint32_t>((size_t)kRadixBins * (p.ntiles ? p.ntiles : 1));
    for (int b = 0; b < 2; ++b) {
        p.kbuf[b] = c.take<uint32_t>((size_t)std::max<uint64_t>(p.n_local, 1));
        p.vbuf[b] = c.take<uint32_t>((size_t)std::max<uint64_t>(p.n_local, 1));
    }
    p.bytes = c.bytes();
    return p;
}

}  // namespace tgl

extern "C" int tgl_tcsr_build_range_workspace(int64_t n_edges, int32_t n_nodes, int add_reverse, int32_t node_lo,
                                              int32_t node_hi, int64_t n_local_stored, size_t* bytes) {
    if (!bytes || n_edges < 0 || n_nodes < 0 || node_lo < 0 || node_hi < node_lo || node_hi > n_nodes ||
        n_local_stored < 0)
        return TGL_EINVAL;
    if ((uint64_t)n_edges * (add_reverse ? 2 : 1) >= (1ull << 32)) return TGL_EINVAL;
    *bytes = plan_range(n_edges, node_hi - node_lo, n_local_stored, add_reverse ? 1 : 0, nullptr).bytes;
    return TGL_OK;
}

extern "C" int tgl_tcsr_build_range(const int32_t* src, const int32_t* dst, const float* ts, const int32_t* eid,
                                    int64_t n_edges, int32_t n_nodes, int add_reverse, int32_t node_lo, int32_t node_hi,
                                    int64_t n_local_stored, int64_t* indptr, int32_t* nbr, float* ts_out,
                                    int32_t* eid_out, void* aux, size_t aux_bytes, void* workspace, size_t ws_bytes,
                                    void* stream, tgl_tcsr** out) {
    NvtxRange nvtx_("tgl_tcsr_build_range");
    if (!out || !indptr || n_edges < 0 || n_nodes < 0 || node_lo < 0 || node_hi < node_lo || node_hi > n_nodes ||
        n_local_stored < 0)
        return TGL_EINVAL;
    *out = nullptr;
    add_reverse = add_reverse ? 1 : 0;
    const uint64_t es = (uint64_t)n_edges * (add_reverse ? 2 : 1);
    if (es >= (1ull << 32)) return TGL_EINVAL;
    if (n_edges > 0 && (!src || !dst || !ts)) return TGL_EINVAL;
    if (n_local_stored > 0 && (!nbr || !ts_out || !eid_out)) return TGL_EINVAL;
    if (!workspace) return TGL_EINVAL;
    int rc = check_device();
    if (rc) return rc;
    const int32_t nl = node_hi - node_lo;
    RangePlan p = plan_range(n_edges, nl, n_local_stored, add_reverse, workspace);
    if (ws_bytes < p.bytes) return TGL_EWORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;

    // K1 over the whole stream (validation) with the range's histogram; K2 -> the local indptr
    if (cudaMemsetAsync(p.err, 0, sizeof(int), st) != cudaSuccess) return TGL_ECUDA;
    if (nl > 0 && cudaMemsetAsync(p.deg, 0, sizeof(uint32_t) * (size_t)nl, st) != cudaSuccess) return TGL_ECUDA;
    if (n_edges > 0) {
        const int64_t blocks = std::min<int64_t>((n_edges + 255) / 256, 148 * 16);
        validate_hist_kernel<<<(unsigned)blocks, 256, 0, st>>>(src, dst, ts, n_edges, n_nodes, add_reverse, node_lo,
                                                                node_hi, p.deg, p.err);
        if (cudaGetLastError() != cudaSuccess) return TGL_ECUDA;
    }
    if (cuda_rc(exclusive_scan<uint32_t, int64_t>(p.deg, indptr, nl, indptr + nl, p.partial, st))) return TGL_ECUDA;
    int herr = 0;
    int64_t total = 0;
    if (cudaMemcpyAsync(&herr, p.err, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(&total, indptr + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return TGL_ECUDA;
    if (herr) return err_bits_to_code(herr);
    if (total != n_local_stored) return TGL_ECAPACITY;  // the caller's E_s of the range is wrong

    // the range's logical edges in stream order, then the stable passes by (owner - lo)
    if (p.n_local > 0) {
        Stream s{src, dst, ts, eid, add_reverse};
        const uint64_t n = p.n_logical;
        const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16);
        range_flag_kernel<<<blocks, 256, 0, st>>>(s, n, node_lo, node_hi, p.flag);
        if (cuda_rc(exclusive_scan<uint32_t, uint32_t>(p.flag, p.pos, (int64_t)n, (uint32_t*)nullptr, p.partial, st)))
            return TGL_ECUDA;
        range_compact_kernel<<<blocks, 256, 0, st>>>(s, n, node_lo, p.flag, p.pos, p.kbuf[1], p.vbuf[1]);
        const uint64_t m = p.n_local;
        const unsigned grid = (unsigned)p.ntiles;
        for (int pass = 0; pass < p.passes; ++pass) {
            const int shift = 8 * pass;
            const int nb = std::min(8, std::max(0, p.bits - shift));
            const uint32_t mask = nb >= 32 ? 0xffffffffu : ((1u << nb) - 1u);
            const bool last = pass == p.passes - 1;
            const uint32_t* kin = p.kbuf[(pass + 1) & 1];
            const uint32_t* vin = p.vbuf[(pass + 1) & 1];
            uint32_t* kout = last ? nullptr : p.kbuf[pass & 1];
            uint32_t* vout = last ? nullptr : p.vbuf[pass & 1];
            radix_upsweep_kernel<kSrcKV><<<grid, kRadixThreads, 0, st>>>(s, kin, m, shift, mask, p.counts, p.ntiles);
            if (cuda_rc(exclusive_scan<uint32_t, uint32_t>(p.counts, p.counts, (int64_t)kRadixBins * p.ntiles,
                                                           (uint32_t*)nullptr, p.partial, st)))
                return TGL_ECUDA;
            if (last)
                radix_downsweep_kernel<kSrcKV, kDstTCSR><<<grid, kRadixThreads, 0, st>>>(
                    s, kin, vin, m, shift, mask, p.counts, p.ntiles, kout, vout, nbr, ts_out, eid_out, nullptr);
            else
                radix_downsweep_kernel<kSrcKV, kDstKV><<<grid, kRadixThreads, 0, st>>>(
                    s, kin, vin, m, shift, mask, p.counts, p.ntiles, kout, vout, nbr, ts_out, eid_out, nullptr);
            if (cudaGetLastError() != cudaSuccess) return TGL_ECUDA;
        }
    }
    if (aux) {
        rc = tgl_tcsr_aux_build(indptr, ts_out, nbr, eid_out, nl, n_local_stored, aux, aux_bytes, stream);
        if (rc) return rc;
    }
    rc = tgl_tcsr_wrap(indptr, nbr, ts_out, eid_out, aux, aux_bytes, nl, n_local_stored, out);
    if (rc) return rc;
    return tgl_tcsr_set_node_base(*out, node_lo);
}

// the global indptr alone (K1 + K2: validation and the degree scan), e.g. to choose the
// edge-balanced node ranges of the node-sharded mode before every rank builds its own range
extern "C" int tgl_tcsr_indptr_workspace(int64_t n_edges, int32_t n_nodes, size_t* bytes) {
    if (!bytes || n_edges < 0 || n_nodes < 0) return TGL_EINVAL;
    Carve c(nullptr);
    c.take<int>(64);
    c.take<uint32_t>((size_t)std::max(n_nodes, 1));
    c.take<uint64_t>(scan_workspace_bytes(n_nodes) / sizeof(uint64_t));
    *bytes = c.bytes();
    return TGL_OK;
}

extern "C" int tgl_tcsr_indptr(const int32_t* src, const int32_t* dst, const float* ts, int64_t n_edges,
                               int32_t n_nodes, int add_reverse, int64_t* indptr, void* workspace, size_t ws_bytes,
                               void* stream) {
    if (!indptr || n_edges < 0 || n_nodes < 0 || !workspace) return TGL_EINVAL;
    if (n_edges > 0 && (!src || !dst || !ts)) return TGL_EINVAL;
    if ((uint64_t)n_edges * (add_reverse ? 2 : 1) >= (1ull << 32)) return TGL_EINVAL;
    size_t need = 0;
    tgl_tcsr_indptr_workspace(n_edges, n_nodes, &need);
    if (ws_bytes < need) return TGL_EWORKSPACE;
    int rc = check_device();
    if (rc) return rc;
    Carve c(workspace);
    int* err = c.take<int>(64);
    uint32_t* deg = c.take<uint32_t>((size_t)std::max(n_nodes, 1));
    uint64_t* partial = c.take<uint64_t>(scan_workspace_bytes(n_nodes) / sizeof(uint64_t));
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(err, 0, sizeof(int), st) != cudaSuccess) return TGL_ECUDA;
    if (n_nodes > 0 && cudaMemsetAsync(deg, 0, sizeof(uint32_t) * (size_t)n_nodes, st) != cudaSuccess) return TGL_ECUDA;
    if (n_edges > 0) {
        const int64_t blocks = std::min<int64_t>((n_edges + 255) / 256, 148 * 16);
        validate_hist_kernel<<<(unsigned)blocks, 256, 0, st>>>(src, dst, ts, n_edges, n_nodes, add_reverse ? 1 : 0, 0,
                                                                n_nodes, deg, err);
        if (cudaGetLastError() != cudaSuccess) return TGL_ECUDA;
    }
    if (cuda_rc(exclusive_scan<uint32_t, int64_t>(deg, indptr, n_nodes, indptr + n_nodes, partial, st)))
        return TGL_ECUDA;
    int herr = 0;
    if (cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return TGL_ECUDA;
    return err_bits_to_code(herr);
}

// ---------------------------------------------------------------------------- K8 shard bucketing
// Node-sharded mode: stable counting sort of the roots by owner shard, the same
// histogram -> scan -> stable-scatter pass as K3 with digit = owner (world <= 256).
namespace tgl {

__global__ void __launch_bounds__(256) owner_kernel(const int32_t* __restrict__ roots, int64_t n,
                                                    const int64_t* __restrict__ splits, int32_t world,
                                                    uint32_t* __restrict__ owner) {
    __shared__ int64_t sp[kRadixBins + 1];
    for (int r = threadIdx.x; r <= world; r += blockDim.x) sp[r] = splits[r];
    __syncthreads();
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = roots[j];
        // owner = last r with splits[r] <= v (out-of-range ids go to the nearest shard, which
        // reports them through its own sampler error word)
        int lo = 0, hi = world;  // search in [0, world)
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (sp[mid] <= v)
                lo = mid;
            else
                hi = mid;
        }
        owner[j] = (uint32_t)lo;
    }
}

__global__ void shard_counts_kernel(const uint32_t* __restrict__ offsets, uint64_t ntiles, int32_t world, uint64_t n,
                                    int64_t* __restrict__ counts) {
    const int r = threadIdx.x;
    if (r >= world) return;
    const uint64_t a = offsets[(uint64_t)r * ntiles];
    const uint64_t b = r + 1 < world ? offsets[(uint64_t)(r + 1) * ntiles] : n;
    counts[r] = (int64_t)(b - a);
}

struct ShardPlan {
    uint64_t ntiles;
    uint32_t* owner;
    uint32_t* counts;
    uint64_t* partial;
    size_t bytes;
};

static ShardPlan plan_shard(int64_t n, void* ws) {
    ShardPlan p;
    p.ntiles = ((uint64_t)n + kRadixTile - 1) / kRadixTile;
    Carve c(ws);
    p.owner = c.take<uint32_t>((size_t)std::max<int64_t>(n, 1));
    p.counts = c.take<uint32_t>((size_t)kRadixBins * std::max<uint64_t>(p.ntiles, 1));
    p.partial = c.take<uint64_t>(scan_workspace_bytes((int64_t)(kRadixBins * p.ntiles)) / sizeof(uint64_t));
    p.bytes = c.bytes();
    return p;
}

}  // namespace tgl

extern "C" int tgl_shard_bucket_workspace(int64_t n_roots, int32_t world, size_t* bytes) {
    if (!bytes || n_roots < 0 || world < 1 || world > kRadixBins) return TGL_EINVAL;
    if ((uint64_t)n_roots >= (1ull << 31)) return TGL_EINVAL;
    *bytes = plan_shard(n_roots, nullptr).bytes;
    return TGL_OK;
}

extern "C" int tgl_shard_bucket(const int32_t* roots, int64_t n_roots, const int64_t* splits, int32_t world,
                                int32_t* perm, int64_t* counts, void* workspace, size_t ws_bytes, void* stream) {
    if (n_roots < 0 || world < 1 || world > kRadixBins || !splits || !counts || !workspace) return TGL_EINVAL;
    if (n_roots > 0 && (!roots || !perm)) return TGL_EINVAL;
    if ((uint64_t)n_roots >= (1ull << 31)) return TGL_EINVAL;
    int rc = check_device();
    if (rc) return rc;
    ShardPlan p = plan_shard(n_roots, workspace);
    if (ws_bytes < p.bytes) return TGL_EWORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    if (n_roots == 0) return cuda_rc(cudaMemsetAsync(counts, 0, sizeof(int64_t) * world, st));
    const int bits = world <= 1 ? 0 : 32 - __builtin_clz((unsigned)(world - 1));
    const uint32_t mask = (1u << bits) - 1u;
    const int64_t blocks = std::min<int64_t>((n_roots + 255) / 256, 148 * 8);
    owner_kernel<<<(unsigned)blocks, 256, 0, st>>>(roots, n_roots, splits, world, p.owner);
    Stream s{nullptr, nullptr, nullptr, nullptr, 0};
    const unsigned grid = (unsigned)p.ntiles;
    radix_upsweep_kernel<kSrcKeys><<<grid, kRadixThreads, 0, st>>>(s, p.owner, (uint64_t)n_roots, 0, mask, p.counts,
                                                                     p.ntiles);
    if (cuda_rc(exclusive_scan<uint32_t, uint32_t>(p.counts, p.counts, (int64_t)kRadixBins * p.ntiles,
                                                   (uint32_t*)nullptr, p.partial, st)))
        return TGL_ECUDA;
    radix_downsweep_kernel<kSrcKeys, kDstPerm><<<grid, kRadixThreads, 0, st>>>(
        s, p.owner, nullptr, (uint64_t)n_roots, 0, mask, p.counts, p.ntiles, nullptr, nullptr, nullptr, nullptr,
        nullptr, perm);
    shard_counts_kernel<<<1, kRadixBins, 0, st>>>(p.counts, p.ntiles, world, (uint64_t)n_roots, counts);
    return cudaGetLastError() == cudaSuccess ? TGL_OK : TGL_ECUDA;
}
