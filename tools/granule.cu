// granule.cu -- what does one scattered small read cost in DRAM bytes on B200, per load flavour?
// Each thread issues U independent 4-byte loads at uniformly random 128-byte-aligned addresses of
// a 32 GB buffer (plus an optional second load 32 / 64 bytes further, same line or the next).
// Run under `ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum` to get the
// DRAM bytes per request of each variant; the program itself prints the access rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/granule tools/granule.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int V>
__device__ __forceinline__ uint32_t ld(const uint32_t* p) {
    uint32_t v;
    if (V == 0) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
    if (V == 1) asm volatile("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    if (V == 2) asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    if (V == 3) asm volatile("ld.global.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
    if (V == 4) asm volatile("ld.global.L2::128B.u32 %0, [%1];" : "=r"(v) : "l"(p));
    if (V == 5) asm volatile("ld.global.L2::256B.u32 %0, [%1];" : "=r"(v) : "l"(p));
    if (V == 6) asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(v) : "l"(p));
    if (V == 7) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
    if (V == 8) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// OFF: byte offset of a second load from the same base (0 = single load)
template <int V, int U, int OFF>
__global__ void __launch_bounds__(256) probe(const uint32_t* __restrict__ buf, uint64_t n_lines, int iters,
                                             uint32_t seed, unsigned long long* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint32_t v[U][2];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t h = hash32(tid * 2654435761u + (uint32_t)(it * U + u) * 40503u + seed);
            const uint64_t c = ((uint64_t)h * n_lines) >> 32;
            const uint32_t* p = buf + c * 32;  // 128-byte line c
            v[u][0] = ld<V>(p);
            v[u][1] = OFF ? ld<V>(p + OFF / 4) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u][0] ^ v[u][1];
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int V, int OFF>
void run(const char* name, const uint32_t* buf, uint64_t bytes, int sms) {
    constexpr int U = 8;
    const uint64_t n_lines = bytes / 128;
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int grid = sms * 8, iters = 16;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    probe<V, U, OFF><<<grid, 256>>>(buf, n_lines, 1, 1, sink);
    cudaEventRecord(a);
    probe<V, U, OFF><<<grid, 256>>>(buf, n_lines, iters, 7, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double req = (double)grid * 256 * iters * U;
    printf("{\"variant\": \"%s\", \"second_load_offset\": %d, \"requests\": %.0f, \"ms\": %.3f, \"Greq_per_s\": %.2f}\n",
           name, OFF, req, ms, req / (ms * 1e-3) / 1e9);
    cudaFree(sink);
}

int main() {
    const uint64_t bytes = 32ull << 30;
    uint32_t* buf;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
    cudaMemset(buf, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 0>("ld.global.nc", buf, bytes, sms);
    run<1, 0>("ld.global", buf, bytes, sms);
    run<2, 0>("ld.global.L1::no_allocate", buf, bytes, sms);
    run<3, 0>("ld.global.L2::64B", buf, bytes, sms);
    run<4, 0>("ld.global.L2::128B", buf, bytes, sms);
    run<5, 0>("ld.global.L2::256B", buf, bytes, sms);
    run<6, 0>("ld.global.cs", buf, bytes, sms);
    run<7, 0>("ld.global.nc.L1::no_allocate.L2::64B", buf, bytes, sms);
    run<8, 0>("ld.global.cg", buf, bytes, sms);
    run<0, 32>("ld.global.nc +32B", buf, bytes, sms);
    run<0, 64>("ld.global.nc +64B", buf, bytes, sms);
    run<0, 128>("ld.global.nc +128B (next line)", buf, bytes, sms);
    run<8, 64>("ld.global.cg +64B", buf, bytes, sms);
    // smaller footprints: L2-resident (32 MB), beyond L2 but few DRAM pages (1 GB)
    run<0, 0>("ld.global.nc 32MB (L2-resident)", buf, 32ull << 20, sms);
    run<0, 0>("ld.global.nc 1GB", buf, 1ull << 30, sms);
    run<3, 0>("ld.global.L2::64B 1GB", buf, 1ull << 30, sms);
    cudaFree(buf);
    return 0;
}
