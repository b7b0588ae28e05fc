// chain.cuh -- internal entry points shared by sample.cu and sharded.cu (not part of the ABI).
#pragma once

#include "common.cuh"

namespace tgl {

// outputs of one snapshot block of a chain (device pointers; ts_edge may be null)
struct ChainOut {
    int64_t* offsets;
    int32_t* nbr;
    int32_t* eid;
    float* dt;
    float* ts_edge;
    int64_t* n_roots_dev;
    int64_t* nnz_dev;
};

// sample.cu: one chain of Alg. 1 over explicit roots / keys / inherited lower bounds
size_t chain_workspace_bytes(int64_t n, int nsb, int k, int strategy);
int sample_chain(const tgl_tcsr* g, int layer, int snap0, int nsb, const int32_t* rn, const float* rt,
                 const uint64_t* rk, const float* rlo, int64_t n, int k, int strategy, float t_s, uint64_t seed,
                 const ChainOut* outs, void* ws, size_t ws_bytes, cudaStream_t st);

// shard.cu: a reply block in bucket order -> original root order (ts_in / ts_out may be null)
size_t unpermute_workspace_bytes(int64_t n);
int unpermute_block(const int32_t* perm, int64_t n, const int32_t* counts_in, const int32_t* nbr_in,
                    const int32_t* eid_in, const float* dt_in, const float* ts_in, int64_t* off_out, int32_t* nbr_out,
                    int32_t* eid_out, float* dt_out, float* ts_out, void* ws, size_t ws_bytes, cudaStream_t st);

}  // namespace tgl
