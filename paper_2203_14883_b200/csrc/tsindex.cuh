// tsindex.cuh -- the atom index over T-CSR timestamps used by the cut search (internal).
//
// The paper locates candidate windows with per-node pointer arrays pt_0..pt_S advanced once per
// epoch (Sec. 3.1).  Pointers are mutable shared state that serialises batches
// (per-node locks); the GPU path is stateless instead: a lower_bound per cut.  HBM serves
// scattered reads in 64-byte atoms (measured with ncu: DRAM bytes = 2 x the requested 32-byte
// sectors for random sector reads), so the unit of cost is one 64-byte, 16-float group.  To make
// a lower_bound cost ~one atom per level instead of ~log2(deg) scattered probes, the build adds
// an implicit 16-ary search tree over the global ts array:
//
//     level l (l = 1..n_levels):  L_l[j] = ts[j * 16^l],   j < ceil(E_s / 16^l)
//
// Sampling positions are GLOBAL multiples of 16^l, so no per-node offsets are stored; a node's
// entries at level l are the multiples of 16^l inside [indptr[v], indptr[v+1]), contiguous in
// L_l.  Between two consecutive multiples of 16^l lie exactly 15 multiples of 16^(l-1): one
// aligned 16-float group (one atom) of L_(l-1).  Size: sum_l E_s / 16^l ~ E_s / 15 floats.
#pragma once

#include "common.cuh"

namespace tgl {

constexpr int kIndexShift = 4;                     // fan-out 16 = one 64-byte group of floats
constexpr int kMaxIndexLevels = 8;                 // 16^8 = 2^32 > E_s

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
        const uint64_t stride = 1ull << (kIndexShift * l);
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

// The sampler's auxiliary ("aux") buffer: [ts atom index | slot records].  A slot record is the
// {ts, nbr, eid} of one T-CSR slot, padded to 16 bytes so that the copy kernel reads it with ONE
// aligned 16-byte load per output: three 4-byte loads per output kept the uniform copy kernel at
// 94 % of its L1 throughput (C4 layer 1, profiles/r02/c4); 12- vs 16-byte records were within
// 2.3 % on C5 runs, which now use the codec's 8-byte packed records.
constexpr int kRecWords = 4;  // {ts, nbr, eid, 0}: 16 bytes
struct SlotRec {
    float ts;
    int32_t nbr;
    int32_t eid;
    int32_t pad;
};
static_assert(sizeof(SlotRec) == 4 * kRecWords, "slot record size");

// Per-node 64-byte record {lo, hi, f[0..13]}: the list bounds and 14 "fences" -- the ts of the
// slots P_j = lo + floor(j (d-1) / 13), j = 0..13 (f[0] = first, f[13] = last edge time; +inf for
// an empty list).  One 64-byte read (one DRAM atom, read by 4 cooperating lanes) gives the bounds
// AND narrows every cut to one gap between consecutive fences: with m = #fences < x, the lower
// bound lies in [P_(m-1) + 1, P_m] -- for d <= 14 the fences are the whole list (no list access at
// all), for d <= 53 at most 3 slots remain (one 64-byte group of ts).
constexpr int kFences = 14;
struct NodeRec {
    uint32_t lo, hi;
    float f[kFences];
};
static_assert(sizeof(NodeRec) == 64, "node record is one 64-byte DRAM atom");

__host__ __device__ inline uint32_t fence_pos(uint32_t lo, uint32_t d, int j) {
    // j (d - 1) < 2^32 for d <= 2^28: one 32-bit multiply-high for the division by 13 (the window
    // kernel runs this 8 times per root); longer lists take the 64-bit path -- same value
    if (d <= (1u << 28)) return lo + ((uint32_t)j * (d - 1u)) / (uint32_t)(kFences - 1);
    return lo + (uint32_t)(((uint64_t)j * (uint64_t)(d - 1)) / (uint64_t)(kFences - 1));
}

// ---------------------------------------------------------------------------- time codes
// When the T-CSR holds at most kMaxCodes distinct timestamps -- MAG's are publication years,
// max(t) = 120 (Table 3) -- the aux build adds a lossless time codec: the sorted
// distinct values value[0..D) (a dictionary) and per slot its code = index of its ts in value[].
// Codes order like the times (ts < x  <=>  code < q(x), q(x) = #{values < x}), so the cut search
// runs on 7-bit codes: a 64-byte node record holds 54 fence codes instead of 14 fence times (gaps
// of d/53 slots instead of d/13), and a 64-byte probe atom covers 64 slots instead of 16.  When the
// widths fit, the slot record shrinks to 8 bytes: nbr | code << bn | (eid - eid_base[code]) << (bn
// + bc); the copy kernel decodes ts = value[code] (the exact stored float) and eid from
// dictionaries in shared memory.  Requests per C5 root (tools/census_c5.py): probes 0.59 -> 0.19,
// selected-record lines 1.01 -> 0.83.
//
// Node record under the codec (16 words): w0 = lo, w1 = hi, w2..w4 = 10 separator codes (+ 2 pad
// bytes), w5..w15 = 11 groups of 4 codes.  Fence j = 5g + r (P_j = lo + floor(j (d-1) / 53)) is
// byte r of group g for r < 4 and separator g for r = 4, so #fences < q = 5 c1 + c2 with c1 =
// #separators < q and c2 = #codes < q in group c1 -- two SWAR byte compares (codes < 128: no
// borrow crosses a byte) instead of a 6-step binary search.  Code 127 (pads, empty lists) is +inf.
constexpr int kMaxCodes = 127;   // 7-bit codes, q(x) <= 127; code 127 = +inf
constexpr int kCodeFences = 54;  // 10 separators + 11 groups of 4
constexpr int kCodeSeps = 10;
constexpr uint32_t kCodeInf = 127u;
constexpr uint32_t kDictMagic = 0x54474344u;  // "TGCD"
// Without the codec (more distinct times), slot records still pack into 8 bytes when every time is
// an integer below 2^24 -- GDELT's 15-minute ticks to 1.8e5 (Table 3) -- and the widths
// fit: packed = 2, {nbr | (eid - eid_base[0]) << bn | time << (bn + be)} with be = bits_code; the
// copy kernel decodes ts = (float)time, exact below 2^24.
struct TimeDict {
    uint32_t magic;
    uint32_t n_codes;    // D (0: no codec: more than kMaxCodes distinct times, or -0 / non-finite)
    uint32_t packed;     // 1: 8-byte records with time codes; 2: 8-byte records with integer times
    uint32_t bits_nbr;   // bn
    uint32_t bits_code;  // bc (packed = 1) / be, the eid offset width (packed = 2)
    int32_t eid_base0;   // packed = 2: the smallest eid
    uint32_t pad[2];
    float value[256];       // sorted distinct timestamps, +inf beyond D
    int32_t eid_base[256];  // smallest eid of each code (packed records)
};
// build scratch behind the dictionary (aux build only)
struct CodecScratch {
    uint32_t hash[512];  // distinct ts bits (open addressing, 0xffffffff = empty)
    int32_t eid_min[256], eid_max[256];
    uint32_t count, overflow, nbr_max, pad;
    uint32_t t_max_bits, not_int;  // integer-time packing: largest time (float bits), any non-integer
    int32_t e_min, e_max;
};
constexpr uint64_t kDictBytes = 8192;
static_assert(sizeof(TimeDict) + sizeof(CodecScratch) <= kDictBytes, "dictionary region");

__host__ __device__ inline uint32_t code_fence_pos(uint32_t lo, uint32_t d, int j) {
    if (d <= (1u << 26)) return lo + ((uint32_t)j * (d - 1u)) / (uint32_t)(kCodeFences - 1);
    return lo + (uint32_t)(((uint64_t)j * (uint64_t)(d - 1)) / (uint64_t)(kCodeFences - 1));
}

struct AuxLayout {
    IndexLayout index;
    uint64_t index_off = 0;  // byte offset of the index levels (after the dictionary region)
    uint64_t rec_off = 0;    // byte offset of the slot records (16-byte SlotRec, or 8-byte packed)
    uint64_t node_off = 0;   // byte offset of the NodeRec array
    uint64_t code_off = 0;   // byte offset of the per-slot time codes (u8)
    uint64_t bytes = 0;
};

inline AuxLayout aux_layout(uint64_t n_stored, uint64_t n_nodes) {
    AuxLayout A;
    A.index = index_layout(n_stored);
    A.index_off = kDictBytes;
    A.rec_off = align_up(A.index_off + A.index.floats * sizeof(float), 256);
    A.node_off = align_up(A.rec_off + n_stored * sizeof(SlotRec), 256);
    A.code_off = align_up(A.node_off + n_nodes * sizeof(NodeRec), 256);
    A.bytes = align_up(A.code_off + n_stored + 64, 256);  // + 64: whole-atom probe reads
    return A;
}

}  // namespace tgl
