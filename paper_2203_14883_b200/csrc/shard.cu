// shard.cu -- node-sharded mode: un-permute the replies of the owners.
//
// The roots of a rank were stably bucketed by owner shard (tgl_shard_bucket, K8) and sent in that
// order; each owner sampled them and sent back one CSR block per snapshot in the same order.
// tgl_shard_unpermute turns such a block (bucket order) into the block the replicated mode would
// have produced (original root order): counts scatter -> exclusive scan -> segmented copy.
#include <algorithm>

#include "chain.cuh"
#include "common.cuh"
#include "scan.cuh"

namespace tgl {

__global__ void unpermute_counts_kernel(const int32_t* __restrict__ perm, int64_t n, const int32_t* __restrict__ cnt_in,
                                        uint32_t* __restrict__ counts_orig) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        counts_orig[perm[j]] = (uint32_t)cnt_in[j];
}

__global__ void offsets_to_counts_kernel(const int64_t* __restrict__ off, int64_t n, int32_t* __restrict__ cnt) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        cnt[j] = (int32_t)(off[j + 1] - off[j]);
}

// one warp per 32 consecutive bucket positions; their source edges are one contiguous range
__global__ void __launch_bounds__(256) unpermute_copy_kernel(const int32_t* __restrict__ perm, int64_t n,
                                                             const int64_t* __restrict__ off_in,
                                                             const int64_t* __restrict__ off_out,
                                                             const int32_t* __restrict__ nbr_in,
                                                             const int32_t* __restrict__ eid_in,
                                                             const float* __restrict__ dt_in, int32_t* __restrict__ nbr_out,
                                                             int32_t* __restrict__ eid_out, float* __restrict__ dt_out,
                                                             const float* __restrict__ ts_in, float* __restrict__ ts_out) {
    __shared__ int64_t s_in[8][33];
    __shared__ int64_t s_dst[8][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t j0 = ((int64_t)blockIdx.x * 8 + warp) * 32;
    if (j0 >= n) return;
    const int64_t j = j0 + lane;
    const int64_t m = n - j0 < 32 ? n - j0 : 32;
    s_in[warp][lane] = j < n ? off_in[j] : off_in[n];
    if (lane == 0) s_in[warp][32] = off_in[j0 + m];
    s_dst[warp][lane] = j < n ? off_out[perm[j]] : 0;
    __syncwarp();
    const int64_t a = s_in[warp][0], b = s_in[warp][32];
    for (int64_t o = a + lane; o < b; o += 32) {
        int r = 0;  // last r with s_in[r] <= o
#pragma unroll
        for (int s2 = 16; s2 > 0; s2 >>= 1)
            if (r + s2 < m && s_in[warp][r + s2] <= o) r += s2;
        const int64_t d = s_dst[warp][r] + (o - s_in[warp][r]);
        nbr_out[d] = nbr_in[o];
        eid_out[d] = eid_in[o];
        dt_out[d] = dt_in[o];
        if (ts_out) ts_out[d] = ts_in[o];
    }
}

struct UnpermPlan {
    uint32_t* counts;
    int64_t* off_in;
    uint64_t* partial;
    size_t bytes;
};

static UnpermPlan plan_unperm(int64_t n, void* ws) {
    UnpermPlan p;
    Carve c(ws);
    p.counts = c.take<uint32_t>((size_t)std::max<int64_t>(n, 1));
    p.off_in = c.take<int64_t>((size_t)n + 1);
    p.partial = c.take<uint64_t>(scan_workspace_bytes(n) / sizeof(uint64_t));
    p.bytes = c.bytes();
    return p;
}

}  // namespace tgl

using namespace tgl;

extern "C" int tgl_shard_unpermute_workspace(int64_t n_roots, size_t* bytes) {
    if (!bytes || n_roots < 0 || n_roots >= (int64_t(1) << 31)) return TGL_EINVAL;
    *bytes = plan_unperm(n_roots, nullptr).bytes;
    return TGL_OK;
}

extern "C" int tgl_offsets_to_counts(const int64_t* offsets, int64_t n_roots, int32_t* counts, void* stream) {
    if (n_roots < 0 || (n_roots > 0 && (!offsets || !counts))) return TGL_EINVAL;
    int rc = check_device();
    if (rc) return rc;
    if (n_roots == 0) return TGL_OK;
    const int64_t blocks = std::min<int64_t>((n_roots + 255) / 256, 148 * 8);
    offsets_to_counts_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(offsets, n_roots, counts);
    return cudaGetLastError() == cudaSuccess ? TGL_OK : TGL_ECUDA;
}

namespace tgl {
size_t unpermute_workspace_bytes(int64_t n) { return plan_unperm(n, nullptr).bytes; }

int unpermute_block(const int32_t* perm, int64_t n_roots, const int32_t* counts_in, const int32_t* nbr_in,
                    const int32_t* eid_in, const float* dt_in, const float* ts_in, int64_t* offsets_out,
                    int32_t* nbr_out, int32_t* eid_out, float* dt_out, float* ts_out, void* workspace,
                    size_t ws_bytes, cudaStream_t st) {
    UnpermPlan p = plan_unperm(n_roots, workspace);
    if (ws_bytes < p.bytes) return TGL_EWORKSPACE;
    if (n_roots == 0) return cuda_rc(cudaMemsetAsync(offsets_out, 0, sizeof(int64_t), st));
    const int64_t blocks = std::min<int64_t>((n_roots + 255) / 256, 148 * 8);
    // bucket-order offsets of the received block, then original-order counts and offsets
    if (cuda_rc(exclusive_scan<int32_t, int64_t>(counts_in, p.off_in, n_roots, p.off_in + n_roots, p.partial, st)))
        return TGL_ECUDA;
    unpermute_counts_kernel<<<(unsigned)blocks, 256, 0, st>>>(perm, n_roots, counts_in, p.counts);
    if (cuda_rc(exclusive_scan<uint32_t, int64_t>(p.counts, offsets_out, n_roots, offsets_out + n_roots, p.partial, st)))
        return TGL_ECUDA;
    const int64_t grid = (n_roots + 255) / 256;
    unpermute_copy_kernel<<<(unsigned)grid, 256, 0, st>>>(perm, n_roots, p.off_in, offsets_out, nbr_in, eid_in, dt_in,
                                                          nbr_out, eid_out, dt_out, ts_out ? ts_in : nullptr, ts_out);
    return cudaGetLastError() == cudaSuccess ? TGL_OK : TGL_ECUDA;
}
}  // namespace tgl

extern "C" int tgl_shard_unpermute(const int32_t* perm, int64_t n_roots, const int32_t* counts_in,
                                   const int32_t* nbr_in, const int32_t* eid_in, const float* dt_in,
                                   int64_t* offsets_out, int32_t* nbr_out, int32_t* eid_out, float* dt_out,
                                   void* workspace, size_t ws_bytes, void* stream) {
    if (n_roots < 0 || n_roots >= (int64_t(1) << 31) || !offsets_out || !workspace) return TGL_EINVAL;
    if (n_roots > 0 && (!perm || !counts_in)) return TGL_EINVAL;
    int rc = check_device();
    if (rc) return rc;
    return unpermute_block(perm, n_roots, counts_in, nbr_in, eid_in, dt_in, nullptr, offsets_out, nbr_out, eid_out,
                           dt_out, nullptr, workspace, ws_bytes, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------- Alg. 2 schedule
// Random chunk scheduling (Alg. 2; R#26): the first batch of epoch
// e starts at e_s = r * cs, r = floor(x * (bs / cs) / 2^32), x = Philox4x32-10 word 0 of counter
// (e_lo, e_hi, 0x414C4732, 0) under key = seed; batch b covers edges [e_s + b bs, e_s + (b+1) bs)
// while its end <= |E|.  One small kernel writes the batch starts and their count on the device.
namespace tgl {
__global__ void chunk_schedule_kernel(int64_t n_edges, int64_t bs, int64_t cs, uint64_t epoch, uint32_t seed_lo,
                                      uint32_t seed_hi, int64_t* __restrict__ first_edge, int64_t cap,
                                      int64_t* __restrict__ n_batches) {
    const uint4 x = philox4x32_10(make_uint4((uint32_t)epoch, (uint32_t)(epoch >> 32), 0x414C4732u, 0u), seed_lo,
                                  seed_hi);
    const int64_t r = (int64_t)(((uint64_t)x.x * (uint64_t)(bs / cs)) >> 32);
    const int64_t e_s = r * cs;
    const int64_t nb = n_edges >= e_s + bs ? (n_edges - e_s) / bs : 0;
    const int64_t m = nb < cap ? nb : cap;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < m; b += (int64_t)gridDim.x * blockDim.x)
        first_edge[b] = e_s + b * bs;
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_batches = nb;
}
}  // namespace tgl

extern "C" int tgl_chunk_schedule(int64_t n_edges, int64_t batch_size, int64_t chunk_size, uint64_t epoch,
                                  uint64_t seed, int64_t* first_edge, int64_t cap, int64_t* n_batches, void* stream) {
    if (n_edges < 0 || batch_size <= 0 || chunk_size <= 0 || chunk_size > batch_size || cap < 0 || !n_batches)
        return TGL_EINVAL;
    if (cap > 0 && !first_edge) return TGL_EINVAL;
    if (cap < n_edges / batch_size) return TGL_ECAPACITY;
    int rc = check_device();
    if (rc) return rc;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((cap + 255) / 256, 148 * 4));
    chunk_schedule_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        n_edges, batch_size, chunk_size, epoch, (uint32_t)seed, (uint32_t)(seed >> 32), first_edge, cap, n_batches);
    return cudaGetLastError() == cudaSuccess ? TGL_OK : TGL_ECUDA;
}

// ---------------------------------------------------------------------------- R#28 validity
namespace tgl {
__global__ void edge_valid_set_kernel(uint32_t* __restrict__ valid, int64_t n_bits, const int32_t* __restrict__ eids,
                                      int64_t n, int32_t value) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = eids[i];
        if (e < 0 || e >= n_bits) continue;
        const uint32_t bit = 1u << (e & 31);
        if (value)
            atomicOr(valid + (e >> 5), bit);
        else
            atomicAnd(valid + (e >> 5), ~bit);
    }
}
}  // namespace tgl

extern "C" int tgl_edge_valid_set(uint32_t* valid, int64_t n_bits, const int32_t* eids, int64_t n, int32_t value,
                                  void* stream) {
    if (n < 0 || n_bits < 0 || (n > 0 && (!valid || !eids)) || (value != 0 && value != 1)) return TGL_EINVAL;
    int rc = check_device();
    if (rc) return rc;
    if (n == 0) return TGL_OK;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 4));
    edge_valid_set_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(valid, n_bits, eids, n, value);
    return cudaGetLastError() == cudaSuccess ? TGL_OK : TGL_ECUDA;
}

// ---------------------------------------------------------------------------- sharded tables
// inv[perm[j]] = j: turns a bucket-order row list back into request order with one tgl_gather
// (node-sharded gather).
namespace tgl {
__global__ void perm_invert_kernel(const int32_t* __restrict__ perm, int64_t n, int32_t* __restrict__ inv) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        inv[perm[j]] = (int32_t)j;
}
}  // namespace tgl

extern "C" int tgl_perm_invert(const int32_t* perm, int64_t n, int32_t* inv, void* stream) {
    if (n < 0 || n >= (int64_t(1) << 31) || (n > 0 && (!perm || !inv))) return TGL_EINVAL;
    int rc = check_device();
    if (rc) return rc;
    if (n == 0) return TGL_OK;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
    perm_invert_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(perm, n, inv);
    return cudaGetLastError() == cudaSuccess ? TGL_OK : TGL_ECUDA;
}
