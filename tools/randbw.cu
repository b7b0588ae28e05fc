// randbw.cu -- calibration microbenchmark for the random-access HBM roofline (SURVEY 8(d)
// "Calibration").  Reads W-byte chunks at uniformly random W-aligned addresses of a buffer of
// GB gigabytes, U independent accesses in flight per thread, and reports the useful bytes/s.
//   mode "thread": each thread reads its own chunk (W/16 LDG.128 from one thread)
//   mode "coop":   W/16 consecutive lanes read one chunk together (one coalesced request)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/randbw tools/randbw.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int W, int U, bool COOP>
__global__ void __launch_bounds__(256) randread(const uint4* __restrict__ buf, uint64_t n_chunks, int iters,
                                                uint32_t seed, unsigned long long* sink) {
    constexpr int V = W >= 16 ? W / 16 : 1;  // uint4 per chunk
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t grp = COOP ? tid / V : tid;   // cooperating lanes share a chunk id
    const int sub = COOP ? (int)(tid % V) : 0;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint4 v[U][COOP ? 1 : V];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t h = hash32(grp * 2654435761u + (uint32_t)(it * U + u) * 40503u + seed);
            const uint64_t c = ((uint64_t)h * n_chunks) >> 32;
            if (W >= 16) {
                if (COOP) v[u][0] = __ldg(buf + c * V + sub);
                else {
#pragma unroll
                    for (int j = 0; j < V; ++j) v[u][j] = __ldg(buf + c * V + j);
                }
            } else {
                const uint32_t* p = reinterpret_cast<const uint32_t*>(buf) + c * (W / 4);
                v[u][0].x = __ldg(p);
                v[u][0].w = 0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < (COOP ? 1 : V); ++j) acc += v[u][j].x ^ v[u][j].w;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

// whole warp reads one W-byte chunk (W multiple of 512) with W/512 coalesced LDG.128 per lane
template <int W, int U>
__global__ void __launch_bounds__(256) warpread(const uint4* __restrict__ buf, uint64_t n_chunks, int iters,
                                                uint32_t seed, unsigned long long* sink) {
    constexpr int R = W / 512;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t wid = tid >> 5, lane = tid & 31;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint4 v[U][R];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t h = hash32(wid * 2654435761u + (uint32_t)(it * U + u) * 40503u + seed);
            const uint64_t c = ((uint64_t)h * n_chunks) >> 32;
#pragma unroll
            for (int r = 0; r < R; ++r) v[u][r] = __ldg(buf + c * (W / 16) + r * 32 + lane);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int r = 0; r < R; ++r) acc += v[u][r].x ^ v[u][r].w;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int W, int U>
void runw(const uint4* buf, uint64_t bytes, int bps, int sms) {
    const uint64_t n_chunks = bytes / W;
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int grid = sms * bps;
    const int iters = 16;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    warpread<W, U><<<grid, 256>>>(buf, n_chunks, 2, 1, sink);
    cudaEventRecord(a);
    warpread<W, U><<<grid, 256>>>(buf, n_chunks, iters, 7, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double chunks = (double)grid * 8 * iters * U;
    printf("  {\"mode\": \"warp\", \"W\": %d, \"U\": %d, \"gb\": %.2f, \"useful_GBps\": %.1f, \"Gaccess_per_s\": %.2f},\n",
           W, U, bytes / 1073741824.0, chunks * W / (ms * 1e-3) / 1e9, chunks / (ms * 1e-3) / 1e9);
    cudaFree(sink);
}

template <int W, int U, bool COOP>
void run(const char* name, const uint4* buf, uint64_t bytes, int bps, int sms) {
    const uint64_t n_chunks = bytes / W;
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int grid = sms * bps;
    const int iters = 32;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    randread<W, U, COOP><<<grid, 256>>>(buf, n_chunks, 2, 1, sink);
    cudaEventRecord(a);
    randread<W, U, COOP><<<grid, 256>>>(buf, n_chunks, iters, 7, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double chunks = (double)grid * 256 / (COOP ? (W >= 16 ? W / 16 : 1) : 1) * iters * U;
    printf("  {\"mode\": \"%s\", \"W\": %d, \"U\": %d, \"gb\": %.2f, \"useful_GBps\": %.1f, \"Gaccess_per_s\": %.2f},\n",
           name, W, U, bytes / 1073741824.0, chunks * W / (ms * 1e-3) / 1e9, chunks / (ms * 1e-3) / 1e9);
    cudaFree(sink);
}

int main(int argc, char** argv) {
    size_t max_gb = argc > 1 ? atoi(argv[1]) : 32;
    uint4* buf;
    if (cudaMalloc(&buf, max_gb << 30) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(buf, 1, max_gb << 30);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("{\"results\": [\n");
    for (double gb : {0.5, 32.0}) {
        if (gb > max_gb) continue;
        const uint64_t bytes = (uint64_t)(gb * 1073741824.0);
        run<4, 8, false>("thread", buf, bytes, 8, sms);
        run<32, 8, false>("thread", buf, bytes, 8, sms);
        run<64, 4, false>("thread", buf, bytes, 8, sms);
        run<32, 8, true>("coop", buf, bytes, 8, sms);
        run<64, 8, true>("coop", buf, bytes, 8, sms);
        run<128, 8, true>("coop", buf, bytes, 8, sms);
        run<16, 8, false>("thread", buf, bytes, 8, sms);
        run<256, 8, true>("coop", buf, bytes, 8, sms);
        runw<512, 4>(buf, bytes, 8, sms);
        runw<1024, 4>(buf, bytes, 8, sms);
        runw<2048, 2>(buf, bytes, 8, sms);
        runw<4096, 2>(buf, bytes, 8, sms);
    }
    printf("  {\"end\": true}\n]}\n");
    cudaFree(buf);
    return 0;
}
