// scan.cuh -- device-wide exclusive scan (reduce / scan-partials / downsweep), used by the
// T-CSR build (K2: degrees -> indptr, "an indptr array of size |V|+1") and by the
// radix passes of the stable scatter (K3).  Internal, not part of the ABI.
#pragma once

#include "common.cuh"

namespace tgl {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096 elements per block

// Block-wide exclusive scan of one uint64 per thread; returns the block total in *total.
__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t v, uint64_t* total, uint64_t* sm /*[33]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint64_t w = lane < nw ? sm[lane] : 0;
        uint64_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(kFull, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < nw) sm[lane] = wi - w;  // exclusive warp offsets
        if (lane == nw - 1) sm[32] = wi;   // block total
    }
    __syncthreads();
    uint64_t r = sm[warp] + x - v;
    *total = sm[32];
    __syncthreads();
    return r;
}

template <typename InT>
__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const InT* __restrict__ in, int64_t n,
                                                                   uint64_t* __restrict__ partial) {
    __shared__ uint64_t sm[33];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint64_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
        if (i < n) s += (uint64_t)in[i];
    }
    uint64_t tot;
    block_excl_scan_u64(s, &tot, sm);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// One block of 1024 threads scans the partials in place (exclusive); writes the grand total
// to *total_out (as OutT) if non-null.
template <typename OutT>
__global__ void __launch_bounds__(1024) scan_partials_kernel(uint64_t* __restrict__ partial, int64_t nb,
                                                             OutT* __restrict__ total_out) {
    __shared__ uint64_t sm[33];
    uint64_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += blockDim.x) {
        int64_t b = b0 + threadIdx.x;
        uint64_t v = b < nb ? partial[b] : 0;
        uint64_t tot;
        uint64_t ex = block_excl_scan_u64(v, &tot, sm);
        if (b < nb) partial[b] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0 && total_out) *total_out = (OutT)carry;
}

// Downsweep: out[i] = partial[block] + exclusive prefix within the block.  Safe in place.  The
// tile is staged through shared memory (padded: element e at e + e/32, conflict-free for both the
// coalesced load and a thread's 16 consecutive elements), so global loads and stores are
// coalesced; the in-tile prefixes go back through the same buffer (32-bit when the tile total
// fits, else stored straight from registers).  Inputs are 32-bit.
template <typename InT, typename OutT>
__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(const InT* in, OutT* out, int64_t n,
                                                                 const uint64_t* __restrict__ partial) {
    static_assert(sizeof(InT) == 4, "32-bit scan inputs");
    __shared__ uint64_t sm[33];
    __shared__ uint32_t s_v[kScanTile + kScanTile / 32];
    const int64_t tile0 = (int64_t)blockIdx.x * kScanTile;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int e = j * kScanThreads + threadIdx.x;
        const int64_t i = tile0 + e;
        s_v[e + (e >> 5)] = i < n ? (uint32_t)in[i] : 0u;
    }
    __syncthreads();
    uint32_t v[kScanItems];
    uint64_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int e = threadIdx.x * kScanItems + j;
        v[j] = s_v[e + (e >> 5)];
        s += v[j];
    }
    uint64_t tot;
    const uint64_t ex = block_excl_scan_u64(s, &tot, sm);  // ends with a barrier: s_v is free
    const uint64_t base = partial[blockIdx.x];
    if (tot < (1ull << 32)) {  // block-uniform
        uint32_t run = (uint32_t)ex;
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            const int e = threadIdx.x * kScanItems + j;
            s_v[e + (e >> 5)] = run;
            run += v[j];
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            const int e = j * kScanThreads + threadIdx.x;
            const int64_t i = tile0 + e;
            if (i < n) out[i] = (OutT)(base + s_v[e + (e >> 5)]);
        }
    } else {
        uint64_t run = base + ex;
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            const int64_t i = tile0 + threadIdx.x * kScanItems + j;
            if (i < n) out[i] = (OutT)run;
            run += v[j];
        }
    }
}

inline size_t scan_workspace_bytes(int64_t n) {
    int64_t nb = (n + kScanTile - 1) / kScanTile;
    return align_up((size_t)(nb > 0 ? nb : 1) * sizeof(uint64_t), 256);
}

// out[i] = sum_{j<i} in[j] for i < n; *total_out = sum (device) if non-null.
template <typename InT, typename OutT>
inline cudaError_t exclusive_scan(const InT* in, OutT* out, int64_t n, OutT* total_out, uint64_t* partial,
                                  cudaStream_t st) {
    if (n <= 0) {
        if (total_out) return cudaMemsetAsync(total_out, 0, sizeof(OutT), st);
        return cudaSuccess;
    }
    int64_t nb = (n + kScanTile - 1) / kScanTile;
    scan_reduce_kernel<InT><<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, partial);
    scan_partials_kernel<OutT><<<1, 1024, 0, st>>>(partial, nb, total_out);
    scan_down_kernel<InT, OutT><<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, n, partial);
    return cudaGetLastError();
}

}  // namespace tgl
