// granule2.cu -- do two loads to the same 128-byte line cost one scattered request or two?
// (DESIGN.md section 4).  tools/granule.cu measured that a second INDEPENDENT load 32 or 64 bytes
// after a first one (same line, in flight together) halves the access rate although DRAM bytes do
// not grow.  This probe separates: same 32-byte sector vs another sector of the line, and a second
// load that DEPENDS on the first (issued after the line has arrived: an L1 hit) vs independent.
// Each thread keeps U chains; every access is a 4-byte ld.global.nc at a random line of 32 GB.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/granule2 tools/granule2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint32_t ldnc(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// MODE 0: one load; 1: + independent load at OFF bytes; 2: + load at OFF bytes issued after the
// first returned (address depends on its value, which is 0x01010101 -> masked to 0)
template <int MODE, int OFF>
__global__ void __launch_bounds__(256) probe(const uint32_t* __restrict__ buf, uint64_t n_lines, int iters,
                                             uint32_t seed, unsigned long long* sink) {
    constexpr int U = 8;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint32_t a[U], b[U];
        const uint32_t* base[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t h = hash32(tid * 2654435761u + (uint32_t)(it * U + u) * 40503u + seed);
            base[u] = buf + (((uint64_t)h * n_lines) >> 32) * 32;
            a[u] = ldnc(base[u]);
            b[u] = MODE == 1 ? ldnc(base[u] + OFF / 4) : 0u;
        }
        if (MODE == 2) {
#pragma unroll
            for (int u = 0; u < U; ++u) b[u] = ldnc(base[u] + OFF / 4 + (a[u] & 0x80000000u ? 1 : 0));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += a[u] ^ b[u];
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int MODE, int OFF>
void run(const char* name, const uint32_t* buf, uint64_t bytes, int sms) {
    const uint64_t n_lines = bytes / 128;
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int grid = sms * 8, iters = 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<MODE, OFF><<<grid, 256>>>(buf, n_lines, 1, 1, sink);
    cudaEventRecord(e0);
    probe<MODE, OFF><<<grid, 256>>>(buf, n_lines, iters, 7, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double acc = (double)grid * 256 * iters * 8;  // logical accesses (first loads)
    printf("{\"variant\": \"%s\", \"accesses\": %.0f, \"ms\": %.3f, \"G_accesses_per_s\": %.2f}\n", name, acc, ms,
           acc / (ms * 1e-3) / 1e9);
    cudaFree(sink);
}

int main() {
    const uint64_t bytes = 32ull << 30;
    uint32_t* buf;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
    cudaMemset(buf, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 0>("one load", buf, bytes, sms);
    run<1, 4>("+ independent, same sector (+4 B)", buf, bytes, sms);
    run<1, 32>("+ independent, next sector (+32 B)", buf, bytes, sms);
    run<1, 64>("+ independent, +64 B", buf, bytes, sms);
    run<2, 4>("+ dependent, same sector (+4 B)", buf, bytes, sms);
    run<2, 32>("+ dependent, next sector (+32 B)", buf, bytes, sms);
    run<2, 64>("+ dependent, +64 B", buf, bytes, sms);
    run<2, 128>("+ dependent, next line (+128 B)", buf, bytes, sms);
    cudaFree(buf);
    return 0;
}
