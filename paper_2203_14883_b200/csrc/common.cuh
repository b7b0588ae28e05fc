// common.cuh -- internal device helpers of libtgl.so (sm_100a).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <cstdio>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include "../../include/tgl.h"

namespace tgl {

constexpr uint32_t kFull = 0xffffffffu;

// Device bounds checks of the sampler's computed indices, compiled in only with -DTGL_BOUNDS (a
// debug build run by the GPU tests: compute-sanitizer is unavailable on the test pool).  A failed
// check prints its line and traps, so the launch fails with a CUDA error.
#ifdef TGL_BOUNDS
#define TGL_CHECK(c)                                                          \
    do {                                                                      \
        if (!(c)) {                                                           \
            printf("TGL_CHECK failed: %s (%s:%d)\n", #c, __FILE__, __LINE__); \
            __trap();                                                         \
        }                                                                     \
    } while (0)
#else
#define TGL_CHECK(c) \
    do {             \
    } while (0)
#endif

// Sticky device error bits (one word per handle / one module-global word for gather).
// Priority when mapping to a code: EINVAL > ERANGE > EUNSORTED (same order as the oracle's
// validation, R#20-R#21).
enum : int { kErrRange = 1, kErrInval = 2, kErrUnsorted = 4 };

inline int err_bits_to_code(int bits) {
    if (bits & kErrInval) return TGL_EINVAL;
    if (bits & kErrRange) return TGL_ERANGE;
    if (bits & kErrUnsorted) return TGL_EUNSORTED;
    return TGL_OK;
}

// Philox4x32-10 (Salmon et al. SC'11), R#6.  Two 32x32->64 multiplies per round.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// NVTX range over a host-side ABI call (header-only NVTX v3: a no-op unless a profiler injects)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator over a caller workspace (256-byte aligned carve-outs).
struct Carve {
    char* base;
    size_t off = 0;
    explicit Carve(void* b) : base(static_cast<char*>(b)) {}
    template <typename T>
    T* take(size_t n) {
        off = align_up(off, 256);
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += n * sizeof(T);
        return p;
    }
    size_t bytes() const { return align_up(off, 256); }
};

// Device-capability gate: the library is compiled for sm_100a only.
int check_device();

// Map the last CUDA error (launch or API) to TGL_ECUDA.
inline int cuda_rc(cudaError_t e) { return e == cudaSuccess ? TGL_OK : TGL_ECUDA; }

// byte-copy vector of 2^VS bytes (row copies of tgl_gather / tgl_state_write)
template <int VS>
struct Vec;
template <> struct Vec<4> { using T = uint4; };
template <> struct Vec<3> { using T = uint2; };
template <> struct Vec<2> { using T = uint32_t; };
template <> struct Vec<1> { using T = uint16_t; };
template <> struct Vec<0> { using T = uint8_t; };

// widest chunk (log2 bytes, <= 4) dividing row_bytes and both base addresses
inline uint32_t vec_shift_for(int64_t row_bytes, const void* a, const void* b) {
    uint32_t vs = 4;
    while (vs > 0 && ((row_bytes & ((1 << vs) - 1)) || (reinterpret_cast<uintptr_t>(a) & ((1 << vs) - 1)) ||
                      (reinterpret_cast<uintptr_t>(b) & ((1 << vs) - 1))))
        --vs;
    return vs;
}

}  // namespace tgl

struct tgl_tcsr {
    const int64_t* indptr;
    const int32_t* nbr;
    const float* ts;
    const int32_t* eid;
    int32_t n_nodes;
    int64_t n_stored;
    int* err_dev;  // sticky device error word of this handle (cudaMalloc at creation)
    int device;
    const float* index;      // 16-ary atom index over ts (tsindex.cuh), or null
    int n_levels;
    uint64_t level_off[12];  // float offset of level l in index (levels <= 8)
    const void* recs;        // slot records {ts, nbr, eid, 0} (16 bytes) or codec-packed (8), or null
    const void* nodes;       // 64-byte node records {lo, hi, 14 fence times | 54 fence codes}, or null
    int64_t node_lo;         // node-sharded handle: global id of local node 0
    // time codec (tsindex.cuh "time codes"): on when n_codes > 0
    const void* dict;        // TimeDict (device): sorted distinct times + per-code eid bases
    const uint8_t* codes;    // per-slot time code
    int n_codes, packed, bits_nbr, bits_code;  // packed: 1 time codes, 2 integer times (tsindex.cuh)
    int eid_base0;                             // packed = 2: the smallest eid
};
