/*
 * tgl_oracle.c -- the PARITY ORACLE for the TGL hot path (arXiv 2203.14883).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2203_14883_b200/,
 * include/, the CUDA library) may include, link or call this file.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg use it.
 * It shares no code, header, constant table or helper with the CUDA path.
 *
 * A plain, slow, single-threaded, obviously-correct C implementation of what the
 * paper's method computes, written from PAPER.md (cited as P:Lnnn) and the readings
 * recorded in DESIGN.md section "Readings" (cited as R#n).  Compile with
 *   gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fexcess-precision=standard
 * so every float operation below is one IEEE-754 binary32 operation, round to
 * nearest even, with gradual underflow (x86-64 SSE; no FMA contraction, no FTZ).
 *
 * Contents (each function cites the passage it follows):
 *   oracle_philox4x32_10     Philox4x32-10 (Salmon et al., SC'11), R#6
 *   oracle_tcsr_build        T-CSR = counting sort of the logical edge stream
 *   oracle_tcsr_count / oracle_tcsr_fill
 *                            the same counting sort split into a count pass and a fill
 *                            pass over stream chunks, optionally restricted to a node
 *                            subset (used for billion-edge configs whose full T-CSR
 *                            is only needed for the sampled roots)
 *   oracle_sample_block      one (layer l, snapshot s) block of Alg. 1, P:L217-L243,
 *                            P:L260-L262 (strategies), P:L267 (no leak); uniform with
 *                            replacement as the variant of DESIGN.md R#24; an optional edge
 *                            validity bitmask (R#28: invalid edges are not candidates)
 *   oracle_gather            out[i] = table[id[i]] byte for byte, Fig. 2 step 2
 *   oracle_state_write       Fig. 2 step 6: node memory / mailbox
 *                            update, events applied one by one in batch order, each
 *                            appended to its node's ring of K most recent slots (R#25)
 *
 * Pins (tests/test_oracle_*.py): Philox known-answer vectors, the Fig. 3 hand example
 * (P:L252), the add_reverse tie example, brute force over the whole logical stream
 * (oracle/brute.py, numpy) on random tiny graphs, numpy stable argsort for the build,
 * invariants (no leak, counts, sortedness, partition of snapshot windows) and the
 * uniform-subset distribution.  Parity pinned for every function; the l>=1 with S>1
 * window reading (R#3) by the hand example tests/golden/r3_hops.json and the brute force.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <math.h>

/* Return codes (the oracle's own numbering; the meaning matches DESIGN.md's table). */
#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_ERANGE (-2)
#define ORC_EUNSORTED (-3)

/* ------------------------------------------------------------------------- */
/* Philox4x32-10, written from Salmon, Moraes, Dror, Shaw, "Parallel random   */
/* numbers: as easy as 1, 2, 3", SC'11.  Round function:                      */
/*   (hi0,lo0) = M0 * c0 ; (hi1,lo1) = M1 * c2                                 */
/*   c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)                              */
/* key schedule k += (W0, W1) between rounds; 10 rounds.                       */
/* ------------------------------------------------------------------------- */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += W0; k1 += W1; }
        uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------------------------------- */
/* Logical edge stream (R#19, R#9, R#10).  Input edges i = 0..E-1 arrive in    */
/* chronological order.  Without reverse edges, logical edge j = i is */
/* (owner src_i, neighbour dst_i, ts_i, eid_i).  With add_reverse, logical     */
/* edges 2i and 2i+1 are src_i->dst_i and dst_i->src_i; both carry ts_i, eid_i.*/
/* eid defaults to the input index i when the caller passes none.              */
/* ------------------------------------------------------------------------- */
static void logical_edge(const int32_t *src, const int32_t *dst, const int32_t *eid,
                         int64_t eid_base, int add_reverse, int64_t j,
                         int32_t *owner, int32_t *nbr, int64_t *i_out, int32_t *eid_out)
{
    int64_t i = add_reverse ? (j / 2) : j;
    int reverse = add_reverse ? (int)(j % 2) : 0;
    *owner = reverse ? dst[i] : src[i];
    *nbr = reverse ? src[i] : dst[i];
    *i_out = i;
    *eid_out = eid ? eid[i] : (int32_t)(eid_base + i);
}

/* Validation, reading R#21 / R#20 and SPEC S:L54: ids in range, ts finite and
 * >= 0 (Table 3 caption P:L331: minimum timestamp is 0), stream chronological. */
static int validate_chunk(const int32_t *src, const int32_t *dst, const float *ts, int64_t n,
                          int32_t n_nodes, float prev_ts, int have_prev)
{
    int range_bad = 0, order_bad = 0, value_bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (src[i] < 0 || src[i] >= n_nodes || dst[i] < 0 || dst[i] >= n_nodes) range_bad = 1;
        if (!isfinite(ts[i]) || ts[i] < 0.0f) value_bad = 1;
        if (i > 0 && ts[i - 1] > ts[i]) order_bad = 1;
        if (i == 0 && have_prev && prev_ts > ts[0]) order_bad = 1;
    }
    if (value_bad) return ORC_EINVAL;
    if (range_bad) return ORC_ERANGE;
    if (order_bad) return ORC_EUNSORTED;
    return ORC_OK;
}

/* Count pass of the counting sort over one chunk of the input stream:
 * deg[v] += number of logical edges owned by v.  If keep != NULL only
 * owners with keep[v] != 0 are counted (restricted oracle for billion-edge configs). */
int oracle_tcsr_count(const int32_t *src, const int32_t *dst, const float *ts, int64_t n_edges,
                      int32_t n_nodes, int add_reverse, const uint8_t *keep,
                      float prev_ts, int have_prev, int64_t *deg)
{
    if (n_nodes < 0 || n_edges < 0) return ORC_EINVAL;
    if (n_edges > 0 && (!src || !dst || !ts)) return ORC_EINVAL;
    int rc = validate_chunk(src, dst, ts, n_edges, n_nodes, prev_ts, have_prev);
    if (rc != ORC_OK) return rc;
    int64_t n_logical = add_reverse ? 2 * n_edges : n_edges;
    for (int64_t j = 0; j < n_logical; ++j) {
        int32_t owner, nb, e; int64_t i;
        logical_edge(src, dst, NULL, 0, add_reverse, j, &owner, &nb, &i, &e);
        if (keep && !keep[owner]) continue;
        deg[owner] += 1;
    }
    return ORC_OK;
}

/* Fill pass: place logical edges, in stream order, at cursor[owner]++ -- the
 * in-order placement step of a counting sort, which is stable, so each node's list
 * keeps stream (= chronological) order and needs no sort.  cursor[v] starts
 * at indptr[v] and is carried across chunks by the caller. */
int oracle_tcsr_fill(const int32_t *src, const int32_t *dst, const float *ts, const int32_t *eid,
                     int64_t eid_base, int64_t n_edges, int32_t n_nodes, int add_reverse,
                     const uint8_t *keep, int64_t *cursor,
                     int32_t *nbr_out, float *ts_out, int32_t *eid_out)
{
    if (n_nodes < 0 || n_edges < 0) return ORC_EINVAL;
    int64_t n_logical = add_reverse ? 2 * n_edges : n_edges;
    for (int64_t j = 0; j < n_logical; ++j) {
        int32_t owner, nb, e; int64_t i;
        logical_edge(src, dst, eid, eid_base, add_reverse, j, &owner, &nb, &i, &e);
        if (keep && !keep[owner]) continue;
        int64_t slot = cursor[owner];
        cursor[owner] = slot + 1;
        nbr_out[slot] = nb;
        ts_out[slot] = ts[i];
        eid_out[slot] = e;
    }
    return ORC_OK;
}

/* Whole-stream T-CSR build: histogram of owner degrees, exclusive
 * prefix sum into indptr (|V|+1 entries), in-order placement.  `cursor` is caller
 * scratch of n_nodes int64 entries. */
int oracle_tcsr_build(const int32_t *src, const int32_t *dst, const float *ts, const int32_t *eid,
                      int64_t n_edges, int32_t n_nodes, int add_reverse,
                      int64_t *indptr, int32_t *nbr_out, float *ts_out, int32_t *eid_out,
                      int64_t *cursor)
{
    if (n_nodes < 0 || n_edges < 0) return ORC_EINVAL;
    for (int32_t v = 0; v < n_nodes; ++v) cursor[v] = 0;      /* deg */
    int rc = oracle_tcsr_count(src, dst, ts, n_edges, n_nodes, add_reverse, NULL, 0.0f, 0, cursor);
    if (rc != ORC_OK) return rc;
    int64_t run = 0;
    for (int32_t v = 0; v < n_nodes; ++v) {                    /* exclusive scan */
        indptr[v] = run;
        run += cursor[v];
    }
    indptr[n_nodes] = run;
    for (int32_t v = 0; v < n_nodes; ++v) cursor[v] = indptr[v];
    return oracle_tcsr_fill(src, dst, ts, eid, 0, n_edges, n_nodes, add_reverse, NULL, cursor,
                            nbr_out, ts_out, eid_out);
}

/* lower_bound: first slot p in [lo, hi) with ts[p] >= x, else hi.  The candidate
 * window of a root is [lower_bound(L), lower_bound(U)), i.e. L <= ts < U (R#2). */
static int64_t lower_bound_f32(const float *ts, int64_t lo, int64_t hi, float x)
{
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (ts[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* ------------------------------------------------------------------------- */
/* One (layer l, snapshot s) block of Alg. 1.                    */
/*                                                                             */
/* Window of root i (R#1, R#2, R#3, R#12):                                      */
/*   l == 0: U = t if s == 0 else t (-) (s (x) t_s);   L = t (-) ((s+1) (x) t_s)  */
/*   l >= 1: U = t (the hop root's own time, TGAT multi-hop, R#4),        */
/*           L = root_lo[i], inherited from its layer-0 ancestor (R#3)            */
/* with (-), (x) single fp32 operations.  S == 1 and t_s = +inf give L = -inf.   */
/* Candidates: slots [a, b) of v's list, a = lower_bound(L), b = lower_bound(U)  */
/* -- every candidate has ts < t, the strict no-leak rule.             */
/* Selection (R#5, R#6, R#13):                                    */
/*   most_recent: the k slots closest to the end pointer, [max(a, b-k), b)        */
/*   uniform:     all of [a, b) if c = b-a <= k; otherwise Floyd's k-subset with   */
/*                Philox draws keyed (seed) and countered (j, l<<16|s, rk_lo, rk_hi),*/
/*                r = floor(x * (m+1) / 2^32), output in ascending slot order.     */
/* Outputs per selected slot p: nbr[p], eid[p], dt = t (-) ts[p]; ts_edge = ts[p];  */
/* child key = rk * k + j (R#7); child lo = L (R#3).  Offsets are the running     */
/* count in root order (the MFG).  Roots with an out-of-range id or a     */
/* non-finite time get count 0 and raise *err (R#20).                            */
/* Returns nnz.                                                                 */
/* ------------------------------------------------------------------------- */
int64_t oracle_sample_block(const int64_t *indptr, const int32_t *nbr, const float *ts, const int32_t *eid,
                            int32_t n_nodes,
                            const int32_t *root_node, const float *root_ts, const uint64_t *root_key,
                            const float *root_lo, int64_t n_roots,
                            int32_t layer, int32_t snapshot, float snapshot_len, int32_t k, int32_t strategy,
                            int32_t replacement, uint64_t seed,
                            int64_t *offsets, int32_t *out_nbr, int32_t *out_eid, float *out_dt,
                            float *out_ts_edge, uint64_t *out_child_key, float *out_child_lo,
                            int32_t *err, uint32_t *pick_scratch /* >= k entries */,
                            const uint32_t *edge_valid, int64_t *cand_scratch /* >= max degree */)
{
    int64_t nnz = 0;
    const uint32_t key[2] = { (uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32) };
    for (int64_t i = 0; i < n_roots; ++i) {
        offsets[i] = nnz;
        int32_t v = root_node[i];
        float t = root_ts[i];
        if (v < 0 || v >= n_nodes) { if (err) *err = ORC_ERANGE; continue; }
        if (!isfinite(t)) { if (err) *err = ORC_EINVAL; continue; }

        float U, L;
        if (layer == 0) {
            U = (snapshot == 0) ? t : t - ((float)snapshot * snapshot_len);
            L = t - ((float)(snapshot + 1) * snapshot_len);
        } else {
            U = t;
            L = root_lo ? root_lo[i] : -INFINITY;
        }
        int64_t lo = indptr[v], hi = indptr[v + 1];
        int64_t a = lower_bound_f32(ts, lo, hi, L);
        int64_t b = lower_bound_f32(ts, lo, hi, U);
        if (b < a) b = a;                 /* cannot happen for L <= U; kept for safety */
        int64_t c = b - a;
        /* R#28: with a validity bitmask over edge ids, the candidates are the
         * window's slots whose edge is valid, in slot order; selection works on their ranks. */
        if (edge_valid) {
            int64_t cv = 0;
            for (int64_t p = a; p < b; ++p) {
                uint32_t e = (uint32_t)eid[p];
                if ((edge_valid[e >> 5] >> (e & 31)) & 1u) cand_scratch[cv++] = p;
            }
            c = cv;
        }
        int64_t n_sel = c < (int64_t)k ? c : (int64_t)k;
        if (strategy == 1 && replacement) n_sel = c > 0 ? (int64_t)k : 0;  /* R#24 */
        uint64_t rk = root_key ? root_key[i] : 0;

        /* positions of the selected slots, ascending */
        if (strategy == 1 && replacement) {
            /* uniform WITH replacement (R#24): k independent draws r_j uniform in [0, c), draw j
             * = Floyd's draw j (R#6: word j mod 4 of the block at counter j / 4); ascending (R#13). */
            for (int32_t j = 0; j < (int32_t)n_sel; ++j) {
                uint32_t ctr[4] = { (uint32_t)j / 4u, ((uint32_t)layer << 16) | (uint32_t)snapshot,
                                    (uint32_t)(rk & 0xFFFFFFFFu), (uint32_t)(rk >> 32) };
                uint32_t x[4];
                oracle_philox4x32_10(ctr, key, x);
                pick_scratch[j] = (uint32_t)(((uint64_t)x[j % 4] * (uint64_t)c) >> 32);
            }
            for (int32_t j = 1; j < (int32_t)n_sel; ++j) {
                uint32_t x = pick_scratch[j];
                int32_t q = j - 1;
                while (q >= 0 && pick_scratch[q] > x) { pick_scratch[q + 1] = pick_scratch[q]; --q; }
                pick_scratch[q + 1] = x;
            }
        } else if (strategy == 0 || c <= (int64_t)k) {
            /* ranks: most_recent -> the last n_sel candidates (closest to the end pointer);
             * uniform with c <= k -> all of them */
            int64_t first = (strategy == 0) ? (c - n_sel) : 0;
            for (int64_t j = 0; j < n_sel; ++j) pick_scratch[j] = (uint32_t)(first + j);
        } else {
            /* Floyd's algorithm: for m = c-k .. c-1 draw r uniform in [0, m]; take r
             * if not yet taken, else take m.  Draw j uses word j mod 4 of the Philox block at
             * counter j / 4 (R#6). */
            for (int32_t j = 0; j < k; ++j) {
                uint32_t m = (uint32_t)(c - k + j);
                uint32_t ctr[4] = { (uint32_t)j / 4u, ((uint32_t)layer << 16) | (uint32_t)snapshot,
                                    (uint32_t)(rk & 0xFFFFFFFFu), (uint32_t)(rk >> 32) };
                uint32_t x[4];
                oracle_philox4x32_10(ctr, key, x);
                uint32_t r = (uint32_t)(((uint64_t)x[j % 4] * ((uint64_t)m + 1)) >> 32);
                int taken = 0;
                for (int32_t q = 0; q < j; ++q) if (pick_scratch[q] == r) { taken = 1; break; }
                pick_scratch[j] = taken ? m : r;
            }
            /* ascending order (insertion sort) */
            for (int32_t j = 1; j < k; ++j) {
                uint32_t x = pick_scratch[j];
                int32_t q = j - 1;
                while (q >= 0 && pick_scratch[q] > x) { pick_scratch[q + 1] = pick_scratch[q]; --q; }
                pick_scratch[q + 1] = x;
            }
        }
        for (int64_t j = 0; j < n_sel; ++j) {
            int64_t p = edge_valid ? cand_scratch[pick_scratch[j]] : a + (int64_t)pick_scratch[j];
            int64_t o = nnz + j;
            out_nbr[o] = nbr[p];
            out_eid[o] = eid[p];
            out_dt[o] = t - ts[p];
            if (out_ts_edge) out_ts_edge[o] = ts[p];
            if (out_child_key) out_child_key[o] = rk * (uint64_t)k + (uint64_t)j;
            if (out_child_lo) out_child_lo[o] = L;
        }
        nnz += n_sel;
    }
    offsets[n_roots] = nnz;
    return nnz;
}

/* Gather (Fig. 2 step 2; D6-D8): out[i] = table[ids[i]] byte for byte.
 * id == -1 gives a zero row; any other out-of-range id gives a zero row and raises
 * *err. */
void oracle_gather(const int32_t *ids, int64_t n_ids, const uint8_t *table, int64_t n_rows,
                   int64_t row_bytes, uint8_t *out, int32_t *err)
{
    for (int64_t i = 0; i < n_ids; ++i) {
        int64_t id = ids[i];
        uint8_t *dst = out + i * row_bytes;
        if (id < 0 || id >= n_rows) {
            memset(dst, 0, (size_t)row_bytes);
            if (id != -1 && err) *err = ORC_ERANGE;
            continue;
        }
        memcpy(dst, table + id * row_bytes, (size_t)row_bytes);
    }
}

/* State write (Fig. 2 step 6: "update the memory and the mailbox for next mini-batch";
 * the mailbox stores "a fixed number of most recent mails"; 1 mail, 10 for APAN).
 * Reading R#25: events i = 0..n-1 are applied one at a time in batch order (a chronological batch,
 * P:L247).  Event i of node v = ids[i] writes its row into slot q = pos[v] of v's ring of K slots
 * (table row (v*K + q), row_bytes bytes; ts_table[v*K + q] = ts[i] when given), then
 * pos[v] = (q + 1) mod K.  K = 1 (node memory; pos may be NULL) is "the last event wins".  An id
 * outside [0, n_nodes) skips the event and raises *err. */
void oracle_state_write(const int32_t *ids, const float *ts, int64_t n, int32_t n_nodes, int32_t K,
                        int32_t *pos, float *ts_table, const uint8_t *rows, int64_t row_bytes,
                        uint8_t *table, int32_t *err)
{
    for (int64_t i = 0; i < n; ++i) {
        int32_t v = ids[i];
        if (v < 0 || v >= n_nodes) { if (err) *err = ORC_ERANGE; continue; }
        int32_t q = (K > 1 && pos) ? pos[v] : 0;
        int64_t slot = (int64_t)v * K + q;
        if (table && rows) memcpy(table + slot * row_bytes, rows + i * row_bytes, (size_t)row_bytes);
        if (ts_table) ts_table[slot] = ts[i];
        if (K > 1 && pos) pos[v] = (q + 1) % K;
    }
}

/* Checksum (test infrastructure, not part of the method): 64-bit FNV-1a over n bytes, continuing
 * from h (pass the basis 0xcbf29ce484222325 to start).  Used to compare per-batch digests of the
 * GPU's blocks with the oracle's blocks; written from the FNV-1a definition
 * (h ^= byte; h *= 0x100000001b3 for every byte), pinned by the published test vectors. */
uint64_t oracle_fnv1a64(const uint8_t *p, int64_t n, uint64_t h)
{
    for (int64_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}
