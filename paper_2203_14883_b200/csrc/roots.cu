// roots.cu -- root staging: the roots of a mini-batch from its positive edges and
// negatives, on the device.
#include <algorithm>

#include "common.cuh"

// A mini-batch arrives as TGL trains on it: positive edges (src_i, dst_i, ts_i) with a negative
// destination neg_i each ("600 positive and 600 negative edges"; "4000 + 4000");
// its roots are the root stream of DESIGN.md R#16: root 3i = src_i, 3i+1 = dst_i, 3i+2 = neg_i, all
// at ts_i.  Expanding on the device moves 16 bytes per 3 roots across PCIe instead of 24.
namespace tgl {

__global__ void batch_roots_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                   const int32_t* __restrict__ neg, const float* __restrict__ ts, int64_t first_root,
                                   int64_t n, int32_t* __restrict__ roots, float* __restrict__ root_ts) {
    const int64_t e0 = first_root / 3;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = first_root + j, e = r / 3 - e0;
        const int w = (int)(r % 3);
        roots[j] = w == 0 ? src[e] : (w == 1 ? dst[e] : neg[e]);
        root_ts[j] = ts[e];
    }
}

}  // namespace tgl

using namespace tgl;

extern "C" int tgl_batch_roots(const int32_t* src, const int32_t* dst, const int32_t* neg, const float* ts,
                               int64_t first_root, int64_t n_roots, int32_t* roots, float* root_ts, void* stream) {
    if (first_root < 0 || n_roots < 0) return TGL_EINVAL;
    if (n_roots == 0) return TGL_OK;
    if (!src || !dst || !neg || !ts || !roots || !root_ts) return TGL_EINVAL;
    const int rc = check_device();
    if (rc) return rc;
    const int64_t blocks = std::min<int64_t>((n_roots + 255) / 256, 148 * 8);
    batch_roots_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(src, dst, neg, ts, first_root, n_roots,
                                                                            roots, root_ts);
    return cuda_rc(cudaGetLastError());
}
