// radix.cuh -- stable LSD counting-sort passes (internal): histogram -> scan -> stable scatter,
// 8 bits per pass, the in-tile stable rank from __match_any_sync.  Used by the T-CSR build (K3,
// build.cu), the node-sharded owner bucketing (K8, build.cu) and the state write (state.cu).
#pragma once

#include "common.cuh"

namespace tgl {

constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixItems = 16;                          // per thread
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 4096 logical edges per tile
constexpr int kRadixBins = 256;

// ---------------------------------------------------------------------------- K3 helpers
struct Stream {
    const int32_t* src;
    const int32_t* dst;
    const float* ts;
    const int32_t* eid;  // may be null -> eid = input index
    int add_reverse;
};

__device__ __forceinline__ uint32_t owner_of(const Stream& s, uint64_t j) {
    if (s.add_reverse) {
        const uint64_t i = j >> 1;
        return (uint32_t)((j & 1) ? s.dst[i] : s.src[i]);
    }
    return (uint32_t)s.src[j];
}

// Source of a pass: the raw edge stream (key = owner, value = logical index j), a (key, value)
// buffer pair from the previous pass, or a key buffer whose values are the identity j.
enum { kSrcStream = 0, kSrcKV = 1, kSrcKeys = 2 };
// Destination: (key, value) buffers, the T-CSR arrays at the final slot, or an int64 permutation.
enum { kDstKV = 0, kDstTCSR = 1, kDstPerm = 2 };

// Index of item r of this thread inside the tile: warp-striped, so that the (round, lane)
// order of a warp is the stream order of its 512 items and warps are in stream order.
__device__ __forceinline__ uint64_t tile_item(uint64_t tile, int warp, int r, int lane) {
    return tile * kRadixTile + (uint64_t)warp * (32 * kRadixItems) + (uint64_t)r * 32 + lane;
}

template <int SRC>
__global__ void __launch_bounds__(kRadixThreads) radix_upsweep_kernel(Stream s, const uint32_t* __restrict__ keys_in,
                                                                      uint64_t n, int shift, uint32_t mask,
                                                                      uint32_t* __restrict__ counts, uint64_t ntiles) {
    __shared__ uint32_t hist[kRadixWarps][kRadixBins];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int b = threadIdx.x; b < kRadixWarps * kRadixBins; b += kRadixThreads) (&hist[0][0])[b] = 0;
    __syncthreads();
    const uint64_t tile = blockIdx.x;
#pragma unroll 4
    for (int r = 0; r < kRadixItems; ++r) {
        const uint64_t j = tile_item(tile, warp, r, lane);
        if (j < n) {
            const uint32_t key = SRC == kSrcStream ? owner_of(s, j) : keys_in[j];
            atomicAdd(&hist[warp][(key >> shift) & mask], 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kRadixBins; b += kRadixThreads) {
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < kRadixWarps; ++w) c += hist[w][b];
        counts[(uint64_t)b * ntiles + tile] = c;  // digit-major: scanning it gives global offsets
    }
}

// Downsweep: stable scatter of the tile.  offsets = exclusive scan of counts (digit-major).
template <int SRC, int DST>
__global__ void __launch_bounds__(kRadixThreads) radix_downsweep_kernel(
    Stream s, const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint64_t n, int shift,
    uint32_t mask, const uint32_t* __restrict__ offsets, uint64_t ntiles, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, int32_t* __restrict__ nbr_out, float* __restrict__ ts_out,
    int32_t* __restrict__ eid_out, int32_t* __restrict__ perm_out) {
    __shared__ uint32_t wcnt[kRadixWarps][kRadixBins];
    __shared__ uint32_t dbase[kRadixBins];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t tile = blockIdx.x;
    for (int b = threadIdx.x; b < kRadixWarps * kRadixBins; b += kRadixThreads) (&wcnt[0][0])[b] = 0;
    for (int b = threadIdx.x; b < kRadixBins; b += kRadixThreads) dbase[b] = offsets[(uint64_t)b * ntiles + tile];
    __syncthreads();

    uint32_t key[kRadixItems], val[kRadixItems], rank[kRadixItems];
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
        const uint64_t j = tile_item(tile, warp, r, lane);
        const bool valid = j < n;
        key[r] = valid ? (SRC == kSrcStream ? owner_of(s, j) : keys_in[j]) : 0u;
        val[r] = valid ? (SRC == kSrcKV ? vals_in[j] : (uint32_t)j) : 0u;
        const uint32_t d = valid ? ((key[r] >> shift) & mask) : (uint32_t)kRadixBins;  // sentinel
        const uint32_t peers = __match_any_sync(kFull, d);
        const int leader = __ffs(peers) - 1;
        uint32_t cnt = 0;
        if (valid) cnt = wcnt[warp][d];
        rank[r] = cnt + __popc(peers & lt);
        __syncwarp();
        if (valid && lane == leader) wcnt[warp][d] = cnt + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kRadixBins; b += kRadixThreads) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kRadixWarps; ++w) {
            const uint32_t c = wcnt[w][b];
            wcnt[w][b] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
        const uint64_t j = tile_item(tile, warp, r, lane);
        if (j >= n) continue;
        const uint32_t d = (key[r] >> shift) & mask;
        const uint64_t pos = (uint64_t)dbase[d] + wcnt[warp][d] + rank[r];
        if (DST == kDstTCSR) {
            const uint64_t lj = val[r];
            const uint64_t i = s.add_reverse ? (lj >> 1) : lj;
            const bool rev = s.add_reverse && (lj & 1);
            nbr_out[pos] = rev ? s.src[i] : s.dst[i];
            ts_out[pos] = s.ts[i];
            eid_out[pos] = s.eid ? s.eid[i] : (int32_t)i;
        } else if (DST == kDstPerm) {
            perm_out[pos] = (int32_t)val[r];
        } else {
            keys_out[pos] = key[r];
            vals_out[pos] = val[r];
        }
    }
}

}  // namespace tgl
