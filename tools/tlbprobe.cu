// tlbprobe.cu -- does page locality matter for random 64-B requests on B200?
//
// randbw.cu measured ~49 G coalesced 64-B random requests/s over a 0.5 GB buffer but ~33 G/s over
// 32 GB: the same DRAM request size, so the difference is address translation (TLB reach) or
// DRAM row locality.  This probe separates the two for the sampler's layout decisions:
//   sweep   64-B requests at random addresses of a buffer of GB gigabytes (0.5 .. max)
//   pair    per logical access two 64-B requests: the first random over the buffer, the second
//           at a random 64-B line within +-R bytes of the first (R = 4 KB .. 1 GB), or fully
//           random (R = 0).  If the second request is cheaper when it shares the first's 2 MB
//           page, a node-major layout (node record next to its slot records) pays.
// Output: JSON lines.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tlbprobe tools/tlbprobe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// 4 lanes x 16 B cooperate on one 64-B line; U independent logical accesses in flight per group
template <int U, bool PAIR>
__global__ void __launch_bounds__(256) probe(const uint4* __restrict__ buf, uint64_t n_lines, uint64_t radius_lines,
                                             int iters, uint32_t seed, unsigned long long* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t grp = tid >> 2;
    const int sub = tid & 3;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint4 v[U][PAIR ? 2 : 1];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t h = hash32(grp * 2654435761u + (uint32_t)(it * U + u) * 40503u + seed);
            const uint64_t c = ((uint64_t)h * n_lines) >> 32;
            v[u][0] = __ldg(buf + c * 4 + sub);
            if (PAIR) {
                const uint32_t h2 = hash32(h ^ 0x9e3779b9u);
                uint64_t c2;
                if (radius_lines == 0) {
                    c2 = ((uint64_t)h2 * n_lines) >> 32;
                } else {
                    const int64_t d = (int64_t)(((uint64_t)h2 * (2 * radius_lines + 1)) >> 32) - (int64_t)radius_lines;
                    int64_t cc = (int64_t)c + d;
                    if (cc < 0) cc = -cc;
                    if (cc >= (int64_t)n_lines) cc = 2 * (int64_t)n_lines - 2 - cc;
                    c2 = (uint64_t)cc;
                }
                v[u][1] = __ldg(buf + c2 * 4 + sub);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < (PAIR ? 2 : 1); ++j) acc += v[u][j].x ^ v[u][j].w;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int U, bool PAIR>
static void run(const char* name, const uint4* buf, uint64_t bytes, uint64_t radius_bytes, int sms) {
    const uint64_t n_lines = bytes / 64;
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int grid = sms * 8, iters = 32;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    probe<U, PAIR><<<grid, 256>>>(buf, n_lines, radius_bytes / 64, 2, 1, sink);
    cudaEventRecord(a);
    probe<U, PAIR><<<grid, 256>>>(buf, n_lines, radius_bytes / 64, iters, 7, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double reqs = (double)grid * 64 * iters * U * (PAIR ? 2 : 1);
    printf("{\"mode\": \"%s\", \"gb\": %.2f, \"radius_bytes\": %llu, \"G_requests_per_s\": %.2f, \"ms\": %.3f}\n", name,
           bytes / 1073741824.0, (unsigned long long)radius_bytes, reqs / (ms * 1e-3) / 1e9, ms);
    cudaFree(sink);
}

int main(int argc, char** argv) {
    const size_t max_gb = argc > 1 ? atoi(argv[1]) : 64;
    uint4* buf;
    if (cudaMalloc(&buf, max_gb << 30) != cudaSuccess) {
        printf("{\"error\": \"alloc failed\"}\n");
        return 1;
    }
    cudaMemset(buf, 1, max_gb << 30);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (double gb : {0.5, 1.0, 2.0, 4.0, 8.0, 16.0, 32.0, 48.0, 64.0, 72.0, 80.0, 88.0, 96.0}) {
        if (gb > max_gb) continue;
        run<8, false>("sweep", buf, (uint64_t)(gb * 1073741824.0), 0, sms);
    }
    const size_t pair_gb = argc > 2 ? atoi(argv[2]) : 32;
    const uint64_t bytes = (pair_gb < max_gb ? pair_gb : max_gb) << 30;
    for (uint64_t r : {0ull, 4096ull, 65536ull, 1ull << 20, 16ull << 20, 256ull << 20, 1ull << 30})
        run<4, true>("pair", buf, bytes, r, sms);
    cudaFree(buf);
    return 0;
}
