// tsindex.cuh -- the sector index over T-CSR timestamps used by the cut search (internal).
//
// The paper locates candidate windows with per-node pointer arrays pt_0..pt_S advanced once per
// epoch (Sec. 3.1).  Pointers are mutable shared state that serialises batches
// (per-node locks); the GPU path is stateless instead: a lower_bound per cut.  To make a
// lower_bound cost ~one 32-byte sector per level instead of ~log2(deg) scattered probes, the
// build adds an implicit 8-ary search tree over the global ts array:
//
//     level l (l = 1..n_levels):  L_l[j] = ts[j * 8^l],   j < ceil(E_s / 8^l)
//
// Sampling positions are GLOBAL multiples of 8^l, so no per-node offsets are stored; a node's
// entries at level l are the multiples of 8^l inside [indptr[v], indptr[v+1]), contiguous in L_l.
// Between two consecutive multiples of 8^l lie exactly 7 multiples of 8^(l-1): one aligned
// 8-float group (one sector) of L_(l-1).  Size: sum_l E_s / 8^l ~ E_s / 7 floats.
#pragma once

#include "common.cuh"

namespace tgl {

constexpr int kMaxIndexLevels = 11;  // 8^11 > 2^32 > E_s

struct IndexLayout {
    int n_levels = 0;
    uint64_t off[kMaxIndexLevels + 1] = {0};  // float offset of level l (1-based) in the buffer
    uint64_t len[kMaxIndexLevels + 1] = {0};
    uint64_t floats = 0;
};

inline IndexLayout index_layout(uint64_t n_stored) {
    IndexLayout L;
    uint64_t o = 0;
    for (int l = 1; l <= kMaxIndexLevels; ++l) {
        const uint64_t stride = 1ull << (3 * l);
        if (stride >= n_stored) break;  // a level needs >= 2 entries to discriminate
        const uint64_t n = (n_stored + stride - 1) / stride;
        L.off[l] = o;
        L.len[l] = n;
        o += (n + 63) / 64 * 64;  // 256-byte aligned levels
        L.n_levels = l;
    }
    L.floats = o;
    return L;
}

}  // namespace tgl
