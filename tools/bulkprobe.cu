// bulkprobe.cu -- scattered reads through the TMA bulk-copy path vs the LSU path on B200
// (DESIGN.md section 4).  tools/granule.cu / granule2.cu: LSU loads of <= 128 bytes at random lines
// of a 32 GB buffer run at ~36 G requests/s, and ANY second load to a line (same or other sector,
// independent or issued after the first returned) costs about a full request: the bound is the
// number of outstanding L1 misses per SM over the loaded DRAM latency, not DRAM bytes.  Does
// cp.async.bulk (issued per thread, completing on an mbarrier, no L1 miss tracking) sustain more
// scattered requests per second?
//   lsu  W bytes per access read by one thread (ld.global.nc.v4 x W/16)
//   bulk W bytes per access copied to shared memory by cp.async.bulk (W = 16 .. 256)
// Each thread keeps U accesses in flight per iteration.  Output: JSON lines.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulkprobe tools/bulkprobe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int W, int U>
__global__ void __launch_bounds__(256) lsu(const uint4* __restrict__ buf, uint64_t n_lines, int iters, uint32_t seed,
                                           unsigned long long* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint4 v[U][W / 16];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t h = hash32(tid * 2654435761u + (uint32_t)(it * U + u) * 40503u + seed);
            const uint4* p = buf + (((uint64_t)h * n_lines) >> 32) * 8;  // 128-byte line
#pragma unroll
            for (int c = 0; c < W / 16; ++c)
                asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u][c].x), "=r"(v[u][c].y), "=r"(v[u][c].z), "=r"(v[u][c].w) : "l"(p + c));
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < W / 16; ++c) acc += v[u][c].x ^ v[u][c].w;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int W, int U>
__global__ void __launch_bounds__(256) bulk(const char* __restrict__ buf, uint64_t n_lines, int iters, uint32_t seed,
                                            unsigned long long* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"((int)blockDim.x));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    unsigned char* mine = sm + (size_t)threadIdx.x * U * W;
    const uint32_t dst0 = (uint32_t)__cvta_generic_to_shared(mine);
    uint32_t acc = 0, phase = 0;
    for (int it = 0; it < iters; ++it) {
        uint64_t st;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;" : "=l"(st) : "r"(b), "r"(U * W) : "memory");
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t h = hash32(tid * 2654435761u + (uint32_t)(it * U + u) * 40503u + seed);
            const char* p = buf + (((uint64_t)h * n_lines) >> 32) * 128;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(dst0 + u * W), "l"(p), "r"(W), "r"(b) : "memory");
        }
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                         : "=r"(done) : "r"(b), "r"(phase) : "memory");
        phase ^= 1;
#pragma unroll
        for (int u = 0; u < U; ++u) acc += *reinterpret_cast<const uint32_t*>(mine + u * W);
        __syncthreads();  // every thread has consumed its slots before the next phase overwrites them
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <bool BULK, int W, int U, int CTAS>
void run(const char* buf, uint64_t bytes, int sms) {
    const uint64_t n_lines = bytes / 128;
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int grid = sms * CTAS, iters = 16;
    const size_t smem = BULK ? (size_t)256 * U * W : 0;
    if (BULK) cudaFuncSetAttribute(bulk<W, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (BULK)
            bulk<W, U><<<grid, 256, smem>>>(buf, n_lines, iters, 7 + rep, sink);
        else
            lsu<W, U><<<grid, 256>>>(reinterpret_cast<const uint4*>(buf), n_lines, iters, 7 + rep, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    const double acc = (double)grid * 256 * iters * U;
    printf("{\"path\": \"%s\", \"bytes\": %d, \"in_flight_per_thread\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, "
           "\"G_accesses_per_s\": %.2f, \"GB_per_s\": %.0f, \"err\": \"%s\"}\n",
           BULK ? "bulk" : "lsu", W, U, CTAS, ms, acc / (ms * 1e-3) / 1e9, acc * W / (ms * 1e-3) / 1e9,
           cudaGetErrorString(err));
    fflush(stdout);
    cudaFree(sink);
}

int main() {
    const uint64_t bytes = 32ull << 30;
    char* buf;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
    cudaMemset(buf, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<false, 16, 8, 8>(buf, bytes, sms);
    run<false, 64, 4, 8>(buf, bytes, sms);
    run<true, 16, 8, 4>(buf, bytes, sms);
    run<true, 32, 8, 4>(buf, bytes, sms);
    run<true, 64, 4, 4>(buf, bytes, sms);
    run<true, 64, 8, 2>(buf, bytes, sms);
    run<true, 128, 4, 2>(buf, bytes, sms);
    run<true, 16, 16, 4>(buf, bytes, sms);
    run<true, 64, 2, 8>(buf, bytes, sms);
    cudaFree(buf);
    return 0;
}
