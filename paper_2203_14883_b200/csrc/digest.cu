// digest.cu -- per-batch 64-bit FNV-1a digests of message-flow blocks ("Parity also
// covers every C4/C5 batch the GPU time includes, checked by a per-batch 64-bit checksum (FNV-1a
// over offsets, nbr, eid and dt bits)").  A verification utility next to the path, not a step of
// it: bench.py digests every timed batch and compares the digests with the oracle's.
//
// FNV-1a is sequential by definition, so one thread owns one batch and walks its bytes in the
// order include/tgl.h fixes.  A thread's loads are sequential in its own range (each 128-byte line
// is fetched once and then hit in L1 by the following 31 word loads).
#include "common.cuh"

namespace tgl {

constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;

__device__ __forceinline__ uint64_t fnv_word(uint64_t h, uint32_t w) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        h ^= (w >> (8 * b)) & 0xffu;
        h *= kFnvPrime;
    }
    return h;
}

__global__ void block_digest_kernel(const int64_t* __restrict__ offsets, const int32_t* __restrict__ nbr,
                                    const int32_t* __restrict__ eid, const float* __restrict__ dt,
                                    const int64_t* __restrict__ bounds, int64_t n_batches, uint64_t* __restrict__ out) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_batches) return;
    const int64_t r0 = bounds[j], r1 = bounds[j + 1];
    const int64_t e0 = offsets[r0], e1 = offsets[r1];
    uint64_t h = kFnvBasis;
    for (int64_t i = r0; i <= r1; ++i) {  // offsets rebased to the batch, int64 little-endian
        const uint64_t o = (uint64_t)(offsets[i] - e0);
        h = fnv_word(h, (uint32_t)o);
        h = fnv_word(h, (uint32_t)(o >> 32));
    }
    for (int64_t e = e0; e < e1; ++e) h = fnv_word(h, (uint32_t)nbr[e]);
    for (int64_t e = e0; e < e1; ++e) h = fnv_word(h, (uint32_t)eid[e]);
    for (int64_t e = e0; e < e1; ++e) h = fnv_word(h, __float_as_uint(dt[e]));
    out[j] = h;
}

}  // namespace tgl

using namespace tgl;

extern "C" int tgl_block_digest(const int64_t* offsets, const int32_t* nbr, const int32_t* eid, const float* dt,
                                const int64_t* bounds, int64_t n_batches, uint64_t* out, void* stream) {
    if (n_batches < 0) return TGL_EINVAL;
    if (n_batches == 0) return TGL_OK;
    if (!offsets || !nbr || !eid || !dt || !bounds || !out) return TGL_EINVAL;
    const int rc = check_device();
    if (rc) return rc;
    const int threads = 64;  // few, long-running threads: spread them over the SMs
    block_digest_kernel<<<(unsigned)((n_batches + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
        offsets, nbr, eid, dt, bounds, n_batches, out);
    return cuda_rc(cudaGetLastError());
}
