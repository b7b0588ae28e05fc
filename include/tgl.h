/*
 * tgl.h -- C ABI of libtgl.so: the TGL hot path (arXiv 2203.14883) on B200 (sm_100a).
 *
 *   tgl_tcsr_build   Temporal-CSR construction         PAPER.md L256-L257 (Sec. 3.1, "The T-CSR
 *                                                      Data Structure"), Fig. 3 (L249-L254)
 *   tgl_sample       parallel temporal sampler         Alg. 1 (L217-L243), Sec. 3.1 "Sampling"
 *                                                      (L260-L262), "Parallel Sampling" (L265-L268)
 *   tgl_gather       mini-batch row gather             Fig. 2 step 2 (L201), node memory / mailbox
 *                                                      (L154-L175, L210), edge features (Table 3)
 *   tgl_state_write  node memory / mailbox update       Fig. 2 step 6 (L201), mailbox of the K
 *                                                      most recent mails (L210, L322)
 *   tgl_shard_*, tgl_sample_sharded, tgl_tcsr_build_range
 *                    node-sharded T-CSR + exchange      (not in the paper)
 *   tgl_chunk_schedule  random chunk scheduling         Alg. 2 (L274-L291)
 *
 * Conventions (every entry point):
 *   - Data pointers are DEVICE pointers unless marked (host).  `stream` is a cudaStream_t passed
 *     as void* (NULL = legacy default stream); all device work is enqueued on it, stream-ordered.
 *   - The caller owns every buffer: inputs, outputs and workspaces.  The library never allocates
 *     device memory on the sampling / gather path.  A tgl_tcsr handle is a small host struct that
 *     BORROWS the caller's T-CSR arrays (they must outlive it) plus one 4-byte device error word
 *     allocated at handle creation.
 *   - Return value: TGL_OK (0) or a negative TGL_E* code.  Nothing throws across the ABI.
 *     Host-checkable argument errors return immediately with no device work enqueued.
 *     Data errors detected on the device by tgl_sample / tgl_gather are STICKY: they never stop
 *     the stream; tgl_check() reads and clears them.  tgl_tcsr_build validates synchronously.
 *   - Element types: node ids and edge ids int32, timestamps float32, CSR offsets int64.
 *     E_s = n_edges * (1 + add_reverse) must be < 2^32; n_nodes < 2^31.
 *   - Floating point: every window bound is one IEEE-754 binary32 op, round-to-nearest-even,
 *     no FMA contraction, no flush-to-zero (R#12), so results are bit-identical to the
 *     CPU oracle.
 *   - Requires a device of compute capability 10.0 (B200, sm_100a): otherwise TGL_ENOTSUP.
 */
#ifndef TGL_H_
#define TGL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define TGL_API __attribute__((visibility("default")))
#else
#define TGL_API
#endif

#define TGL_ABI_VERSION 3

enum {
    TGL_OK = 0,
    TGL_EINVAL = -1,     /* bad argument: NULL pointer, L<1, S<1, S>TGL_MAX_SNAPSHOTS, k<1 or
                            k>TGL_MAX_FANOUT, S>1 with non-finite snapshot_len, E_s >= 2^32,
                            V >= 2^31; device-detected: non-finite or negative edge time at build,
                            non-finite root time at sampling (R#20, R#21) */
    TGL_ERANGE = -2,     /* node / row id out of range (device-detected) */
    TGL_EUNSORTED = -3,  /* build input not chronological (device-detected) */
    TGL_ECAPACITY = -4,  /* an output buffer is smaller than tgl_sample_capacity() says */
    TGL_EWORKSPACE = -5, /* workspace smaller than the *_workspace() query says */
    TGL_ECUDA = -6,      /* CUDA runtime error (launch failure, ...) */
    TGL_ENCCL = -7,      /* collective failure (NCCL) in the node-sharded mode */
    TGL_ENOTSUP = -8     /* device is not sm_100 */
};

#define TGL_MAX_SNAPSHOTS 16
#define TGL_MAX_FANOUT 1024
#define TGL_MAX_GATHER_TABLES 8

typedef struct tgl_tcsr tgl_tcsr; /* opaque, host-side */

typedef enum { TGL_MOST_RECENT = 0, TGL_UNIFORM = 1 } tgl_strategy;

TGL_API int tgl_abi_version(void);
TGL_API const char *tgl_strerror(int code);

/* ------------------------------------------------------------------ T-CSR */

/* Bytes of device workspace tgl_tcsr_build needs (host query, no device work). */
TGL_API int tgl_tcsr_build_workspace(int64_t n_edges, int32_t n_nodes, int add_reverse,
                             size_t *bytes /* host, out */);

/*
 * Build the T-CSR of a chronological edge stream.
 *
 * Inputs (device): src[n_edges], dst[n_edges] int32 in [0, n_nodes); ts[n_edges] float32,
 *   finite, >= 0, non-decreasing (the stream is chronological); eid[n_edges] int32 or
 *   NULL (NULL -> eid_i = i).
 * Logical edge stream (R#19): add_reverse = 0 -> logical edge i = (owner src_i, neighbour dst_i);
 *   add_reverse = 1 -> logical edges 2i = src_i->dst_i and 2i+1 = dst_i->src_i, both with
 *   ts_i and eid_i.  E_s = n_edges * (1 + add_reverse).
 * Outputs (device, caller-allocated): indptr[n_nodes+1] int64 (exclusive scan of owner degrees),
 *   nbr[E_s] int32, ts_out[E_s] float32, eid_out[E_s] int32: the logical edges grouped by owner,
 *   each node's list in stream order -- hence time-sorted without a sort -- with ties
 *   broken by stream order (R#8).  Bit-identical to the oracle's counting sort.
 *   ts_out must be 64-byte aligned and its allocation must extend to round_up(E_s, 16) floats: the
 *   sampler reads timestamps in aligned 16-float (64-byte, one HBM atom) groups.
 * aux (optional, may be NULL): >= tgl_tcsr_aux_bytes(E_s, V) bytes, 256-byte aligned; filled with
 *   the sampler's acceleration structures over the T-CSR: the 16-ary index over ts_out (long-list
 *   cut search), a 16-byte record {ts, nbr, eid, 0} per slot (payload copy: one load per output)
 *   and a 64-byte record {lo, hi, 14 fence times} per node (list bounds and cut gaps in one
 *   load) -- DESIGN.md "Data layout".  Without it the sampler reads the separate arrays.
 *   Time codec: when the T-CSR holds at most 127 distinct timestamps (all finite, >= +0; e.g.
 *   MAG's publication years, P:L336 / P:L355) the aux build also writes a dictionary of the
 *   sorted distinct times and a 7-bit code per slot; node records then carry 54 fence codes and,
 *   when nbr / code / per-code eid offset fit 64 bits, slot records shrink to 8 bytes.  Without
 *   codes, slot records still shrink to 8 bytes when every time is an integer below 2^24 and nbr /
 *   eid offset / time fit 64 bits (e.g. GDELT's 15-minute ticks).  Lossless: sampled blocks are
 *   bit-identical with and without either form (tgl_tcsr_codec reports them).
 *   The aux build blocks on `stream` (it reads the distinct-time count and the codec widths).
 * workspace: >= tgl_tcsr_build_workspace() bytes of device memory, 256-byte aligned.
 * Synchronous validation: the call blocks on `stream` once to read the device validation word;
 *   on ERANGE / EINVAL / EUNSORTED no handle is returned and outputs are unspecified.
 * On success *out (host) receives a handle that borrows indptr/nbr/ts_out/eid_out/aux.
 */
TGL_API int tgl_tcsr_build(const int32_t *src, const int32_t *dst, const float *ts, const int32_t *eid,
                   int64_t n_edges, int32_t n_nodes, int add_reverse,
                   int64_t *indptr, int32_t *nbr, float *ts_out, int32_t *eid_out,
                   void *aux, size_t aux_bytes,
                   void *workspace, size_t ws_bytes, void *stream, tgl_tcsr **out /* host */);

/* Bytes of the optional sampler aux buffer for a T-CSR of n_stored edges over n_nodes nodes. */
TGL_API int tgl_tcsr_aux_bytes(int64_t n_stored, int32_t n_nodes, size_t *bytes /* host */);

/* (Re)build the aux buffer over existing T-CSR arrays (e.g. ones received from another rank).
 * Blocks on `stream` (codec detection); the buffer is complete when the call returns. */
TGL_API int tgl_tcsr_aux_build(const int64_t *indptr, const float *ts, const int32_t *nbr, const int32_t *eid,
                       int32_t n_nodes, int64_t n_stored, void *aux, size_t aux_bytes, void *stream);

/* Wrap already-built T-CSR arrays (e.g. received from another rank) in a handle.  No
 * validation beyond NULL / size checks.  n_stored = E_s = indptr[n_nodes].  aux may be NULL or a
 * buffer filled by tgl_tcsr_build / tgl_tcsr_aux_build over the same arrays. */
TGL_API int tgl_tcsr_wrap(const int64_t *indptr, const int32_t *nbr, const float *ts, const int32_t *eid,
                  const void *aux, size_t aux_bytes,
                  int32_t n_nodes, int64_t n_stored, tgl_tcsr **out /* host */);

TGL_API int tgl_tcsr_destroy(tgl_tcsr *g);

/* Node-sharded handles: the handle's T-CSR holds the lists of global nodes
 * [node_lo, node_lo + n_nodes); roots passed to tgl_sample are GLOBAL ids, translated in-kernel
 * (roots outside the range: count 0 + sticky ERANGE).  Neighbour ids stored in the lists stay global. */
TGL_API int tgl_tcsr_set_node_base(tgl_tcsr *g, int64_t node_lo);

/* Host query of a handle's sizes. */
TGL_API int tgl_tcsr_info(const tgl_tcsr *g, int32_t *n_nodes /* host */, int64_t *n_stored /* host */);

/* Host query of the handle's time codec (tgl_tcsr_build "aux"): *n_codes = number of distinct
 * timestamps coded (0: no codec -- no aux, more than 127 distinct times, or -0.0 present);
 * *packed = 1 when slot records are the 8-byte form with time codes, 2 when they are the 8-byte form
 * with integer times (no time codes: every time an integer below 2^24, e.g. GDELT's 15-minute ticks,
 * and nbr / eid offset / time widths fit 64 bits), 0 otherwise.  Either pointer may be NULL. */
TGL_API int tgl_tcsr_codec(const tgl_tcsr *g, int32_t *n_codes /* host */, int32_t *packed /* host */);

/* ------------------------------------------------------------------ sampler (Alg. 1) */

/*
 * One (layer l, snapshot s) message-flow block (the MFG of P:L268), CSR by destination root.
 * Block (l, s) lives at out[l*S + s].  Its destination side (roots) is the caller's roots for
 * l = 0 and block (l-1, s)'s (nbr, ts_edge) in output order for l >= 1 (Alg. 1, R#3, R#4,
 * no dedup R#14).  For root r: edges offsets[r] .. offsets[r+1]-1, in ascending slot (= time)
 * order (R#13), each (nbr = source node, eid, dt = t_root (-) t_edge).
 * The caller allocates every array with the capacities tgl_sample_capacity() reports and sets
 * cap_roots / cap_edges; the library writes n_roots_dev / nnz_dev (device scalars), so no host
 * synchronisation is needed between layers.
 */
typedef struct {
    int64_t cap_roots;    /* in: capacity of offsets is cap_roots + 1 */
    int64_t cap_edges;    /* in: capacity of nbr / eid / dt / ts_edge */
    int64_t *offsets;     /* [n_roots + 1] int64 */
    int32_t *nbr;         /* [nnz] sampled neighbour (MFG source node) */
    int32_t *eid;         /* [nnz] edge id of the sampled temporal edge */
    float *dt;            /* [nnz] t_root (-) t_edge, fp32, > 0 (no leak) */
    float *ts_edge;       /* [nnz] t_edge; REQUIRED when l < L-1 (next layer's root times), else
                             may be NULL (then not written) */
    int64_t *n_roots_dev; /* out: device scalar, number of destination roots of this block */
    int64_t *nnz_dev;     /* out: device scalar, number of sampled edges of this block */
} tgl_block;

/*
 * Capacities for tgl_sample (host query): roots_cap[l] = n_roots * prod_{j<l} fanouts[j],
 * edges_cap[l] = roots_cap[l] * fanouts[l] (per block), and the workspace bytes.
 */
TGL_API int tgl_sample_capacity(int64_t n_roots, int32_t n_layers, const int32_t *fanouts /* host [L] */,
                        int32_t n_snapshots, tgl_strategy strategy, float snapshot_len,
                        int64_t *roots_cap /* host [L] */, int64_t *edges_cap /* host [L] */,
                        size_t *ws_bytes /* host */);

/*
 * Alg. 1 over n_roots roots (node roots[i], time root_ts[i]), L = n_layers layers with fanouts
 * k_l, S = n_snapshots dynamic snapshots of length snapshot_len (+INFINITY allowed iff S == 1).
 *
 * Window of a root (R#1-R#3, R#12):  l = 0: U_s = t (s = 0) or t (-) (s (x) t_s),
 *   L_s = t (-) ((s+1) (x) t_s);  l >= 1: U = the hop root's own time, L inherited.
 *   Candidates = slots of the node's list with L <= ts < U (strictly before the root).
 * Selection (R#5, R#6): TGL_MOST_RECENT -> the min(k, c) latest candidates;
 *   TGL_UNIFORM -> all candidates if c <= k, else Floyd's k-subset drawn with Philox4x32-10,
 *   key (seed_lo, seed_hi), counter (j, l<<16|s, rk_lo, rk_hi), rk = root key (R#7):
 *   root_key_base + i at layer 0, parent_key * k_l + j below.  Per-batch and many-batch calls
 *   therefore give identical bits when root_key_base is the roots' global index.
 * Device-detected errors (out-of-range root id -> ERANGE, non-finite root time -> EINVAL) give
 *   that root a count of 0 and set the sticky word read by tgl_check(g, ...).
 * workspace: >= ws_bytes from tgl_sample_capacity(), device memory, 256-byte aligned, not
 *   shared by concurrent calls.  Launches: one memset, then two kernels (window, copy) per chain:
 *   layer 0 is one chain covering all S snapshots of a root; l >= 1 one chain per snapshot.
 */
TGL_API int tgl_sample(const tgl_tcsr *g, const int32_t *roots, const float *root_ts, int64_t n_roots,
               int32_t n_layers, const int32_t *fanouts /* host [L] */, tgl_strategy strategy,
               int32_t n_snapshots, float snapshot_len, uint64_t seed, uint64_t root_key_base,
               tgl_block *out /* host [L*S] */, void *workspace, size_t ws_bytes, void *stream);

/*
 * tgl_sample with EXPLICIT layer-0 root keys (device uint64 [n_roots]) instead of root_key_base + i:
 * used by the node-sharded mode, where an owner samples roots gathered from many ranks and must
 * reproduce exactly the keys the replicated mode would have used (R#7).  Same semantics otherwise.
 */
TGL_API int tgl_sample_keyed(const tgl_tcsr *g, const int32_t *roots, const float *root_ts,
                     const uint64_t *root_keys, int64_t n_roots, int32_t n_layers,
                     const int32_t *fanouts /* host [L] */, tgl_strategy strategy, int32_t n_snapshots,
                     float snapshot_len, uint64_t seed, tgl_block *out /* host [L*S] */,
                     void *workspace, size_t ws_bytes, void *stream);

/*
 * Sampler variants (the other samplers the paper benchmarks; R#23,
 * R#24).  tgl_sample_ex = tgl_sample / tgl_sample_keyed plus an options struct:
 *   hop_time     TGL_HOP_EDGE_TIME (default, R#4): a hop root's time is its sampled edge's time;
 *                TGL_HOP_ROOT_TIME (R#23): it is its parent root's time, so every layer samples
 *                relative to the layer-0 root's time ("others use the root's timestamp");
 *                dt of layer l >= 1 is then root time (-) edge time.
 *   replacement  TGL_UNIFORM only.  0 (default): without replacement (Floyd, R#5).  1 (R#24): a
 *                root with c > 0 candidates gets exactly k draws r_j = floor(x_j c / 2^32), x_j
 *                from the Philox counter of Floyd's draw j (R#6), output ascending (duplicates
 *                kept); c = 0 gives none.
 *   reserved     must be zero.
 * root_keys: NULL -> root_key_base + i (as tgl_sample), else explicit keys (as tgl_sample_keyed).
 * opts: host pointer or NULL (all defaults).  Errors: TGL_EINVAL for an unknown hop_time,
 * replacement != 0 with TGL_MOST_RECENT, dedup without dedup blocks, or non-zero reserved words;
 * otherwise as tgl_sample.  The workspace size of tgl_sample_capacity() covers hop_time and
 * replacement; dedup needs tgl_sample_capacity_ex().
 */
typedef enum { TGL_HOP_EDGE_TIME = 0, TGL_HOP_ROOT_TIME = 1 } tgl_hop_time;
typedef struct {
    int32_t hop_time;     /* tgl_hop_time */
    int32_t replacement;  /* 0 or 1 */
    int32_t dedup;        /* 0 or 1: per-block distinct (node, hop time) lists (R#27), see below */
    int32_t reserved[5];
    const uint32_t *edge_valid; /* device bitmask over edge ids (bit e of word e/32; R#28) or NULL:
                                   an edge whose bit is 0 is not a candidate ("invalid edges could
                                   be simply ignored"); maintained by tgl_edge_valid_set */
    const struct tgl_fused_gather *gather; /* host pointer or NULL: fused gather of the last layer's
                                   outputs (see tgl_fused_gather below; ABI version 2) */
} tgl_sample_options;

/*
 * Fused gather (Fig. 2 step 2): while the copy kernel writes the
 * last layer's block, it also fills, for every output i of that block, out_t[i] = table_t[id] with
 * id = the output's source node (nbr[i]; node memory, mailbox, their timestamps) or its edge id
 * (eid[i]; edge features) -- the rows of tgl_gather without a second pass over the block.  Rows
 * that are a multiple of 16 bytes (and 16-byte aligned) are copied by a warp per row, narrower
 * ones lane per row (4-byte multiples).  An id outside [0, n_rows) gives a zero row and, unless -1,
 * the sticky ERANGE of the handle.  Supported when the last layer has ONE block (n_snapshots == 1)
 * and without edge validity or dedup (TGL_EINVAL otherwise); out_t needs >= edges_cap[L-1] rows.
 */
#define TGL_MAX_FUSED_GATHER 8
typedef struct {
    const void *table; /* device [n_rows * row_bytes] */
    int64_t n_rows;
    int64_t row_bytes; /* > 0, a multiple of 4 */
    void *out;         /* device [edges_cap * row_bytes], row i = output i of the block */
    int32_t by_edge;   /* 0: rows of the source node (nbr), 1: rows of the edge (eid) */
} tgl_fused_table;
typedef struct tgl_fused_gather {
    int32_t n_tables;  /* 1 .. TGL_MAX_FUSED_GATHER */
    tgl_fused_table tables[TGL_MAX_FUSED_GATHER];
} tgl_fused_gather;

/*
 * dedup = 1 (R#27, SPEC's message-flow-graph node lists): for every block (l, s) the library also
 * writes, into dedup[l*S + s], the distinct (node, hop time) pairs of the block's outputs in order
 * of first appearance (hop time = ts_edge, or the root time under TGL_HOP_ROOT_TIME; equality on
 * the fp32 bit pattern), src_index[i] = the pair of output i, and *n_uniq_dev.  Layer l+1 then
 * samples only those pairs, each with its first occurrence's key (R#7): no redundant sampling or
 * gathering of repeated (node, time) roots.  Requires ts_edge for every layer (edge-time mode) and
 * is not defined for L > 1 with a finite snapshot length (TGL_EINVAL): inherited windows differ.
 * The workspace must come from tgl_sample_capacity_ex() with the same options.
 */
typedef struct {
    int64_t cap;            /* in: >= edges_cap[l] */
    int32_t *src_index;     /* [nnz] index of output i's pair in uniq_* */
    int32_t *uniq_node;     /* [n_uniq] */
    float *uniq_ts;         /* [n_uniq] */
    int64_t *n_uniq_dev;    /* out: device scalar */
} tgl_dedup_block;

TGL_API int tgl_sample_capacity_ex(int64_t n_roots, int32_t n_layers, const int32_t *fanouts /* host [L] */,
                           int32_t n_snapshots, tgl_strategy strategy, float snapshot_len,
                           const tgl_sample_options *opts /* host or NULL */, int64_t *roots_cap /* host [L] */,
                           int64_t *edges_cap /* host [L] */, size_t *ws_bytes /* host */);

TGL_API int tgl_sample_ex(const tgl_tcsr *g, const int32_t *roots, const float *root_ts,
                  const uint64_t *root_keys /* device [n_roots] or NULL */, int64_t n_roots, int32_t n_layers,
                  const int32_t *fanouts /* host [L] */, tgl_strategy strategy, int32_t n_snapshots,
                  float snapshot_len, uint64_t seed, uint64_t root_key_base,
                  const tgl_sample_options *opts /* host or NULL */, tgl_block *out /* host [L*S] */,
                  const tgl_dedup_block *dedup /* host [L*S], required iff opts->dedup */,
                  void *workspace, size_t ws_bytes, void *stream);

/*
 * Edge-validity events (R#28): set (value = 1) or clear (value = 0) the bits of the
 * n edge ids eids[] in the bitmask valid (device uint32 [ceil(E/32)]), e.g. after a mini-batch
 * whose events delete or re-insert edges.  Out-of-range ids are the caller's responsibility
 * (n_bits bounds them: ids >= n_bits are skipped).
 */
TGL_API int tgl_edge_valid_set(uint32_t *valid, int64_t n_bits, const int32_t *eids, int64_t n, int32_t value,
                       void *stream);

/* ------------------------------------------------------------------ gather (Fig. 2 step 2) */

/* One gather target: out row i = table row ids[i]; row_bytes bytes per row. */
typedef struct {
    const void *table; /* device [n_rows * row_bytes] */
    int64_t n_rows;
    int64_t row_bytes;
    void *out;         /* device [n_ids * row_bytes] */
} tgl_gather_table;

/*
 * For every table t and every i < n_ids: out_t[i] = table_t[ids[i]] byte for byte (node memory,
 * mailbox, their timestamps, edge features -- P:L201, L210, Table 3).  id == -1 gives a zero row;
 * any other id outside [0, n_rows) gives a zero row and sets the sticky ERANGE word.
 * n_ids = *n_ids_dev (device scalar, clamped to n_ids_cap) when n_ids_dev != NULL, else
 * n_ids_cap -- so a gather can follow tgl_sample on the stream with no host sync.
 * One kernel launch for all tables (<= TGL_MAX_GATHER_TABLES).
 */
TGL_API int tgl_gather(const int32_t *ids, int64_t n_ids_cap, const int64_t *n_ids_dev,
               const tgl_gather_table *tables /* host [n_tables] */, int32_t n_tables, void *stream);

/* ------------------------------------------------------------------ state write (Fig. 2 step 6) */

/* One state table: rows of the n events (rows[i], row_bytes each) scattered into the node table
 * laid out as n_nodes x K slots of row_bytes (slot q of node v at byte (v*K + q) * row_bytes). */
typedef struct {
    const void *rows;   /* device [n_events * row_bytes] */
    int64_t row_bytes;  /* > 0 */
    void *table;        /* device [n_nodes * K * row_bytes], updated in place */
} tgl_state_table;

/*
 * "Update the memory and the mailbox for next mini-batch" (Fig. 2 step 6, L201; the mailbox keeps
 * "a fixed number of most recent mails", L210; 1 mail, 10 for APAN, L322), reading R#25: the
 * result equals applying events i = 0..n_events-1 one at a time in batch order: event i of node
 * v = ids[i] writes rows_t[i] into slot q = pos[v] of v's ring in every table t, ts[i] into
 * ts_table[v*K + q] (if ts_table != NULL), then pos[v] = (q + 1) mod K.
 *   K = 1: node memory / mem_ts / a 1-mail mailbox -- the last event of each node wins; pos may
 *          be NULL (and is not touched).  K > 1: pos (device int32 [n_nodes], caller-owned ring
 *          cursors, values in [0, K)) is required.
 * Deterministic (no atomic decides a value): a stable sort groups each node's events, only its
 * last K survive, each into a distinct slot.  Device-detected errors: an id outside [0, n_nodes)
 * skips that event and sets the sticky ERANGE word read by tgl_check(NULL, ...).
 * Errors: TGL_EINVAL for K < 1, n_events >= 2^31, K > 1 without pos, a NULL row / table pointer,
 * row_bytes <= 0 or n_tables > TGL_MAX_GATHER_TABLES; TGL_EWORKSPACE if ws_bytes is too small.
 * workspace >= tgl_state_write_workspace() bytes (device, not shared by concurrent calls).
 */
TGL_API int tgl_state_write_workspace(int64_t n_events, int32_t n_nodes, size_t *bytes /* host */);
TGL_API int tgl_state_write(const int32_t *ids, const float *ts, int64_t n_events, int32_t n_nodes, int32_t K,
                    int32_t *pos, float *ts_table, const tgl_state_table *tables /* host [n_tables] */,
                    int32_t n_tables, void *workspace, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ training schedule (Alg. 2) */

/*
 * Random chunk scheduling (Alg. 2), reading R#26: the mini-batches of epoch `epoch`
 * over the chronological training edges [0, n_edges).  The first batch starts at e_s = r * cs,
 * r = floor(x * (bs / cs) / 2^32) with x = Philox4x32-10 word 0 of counter (epoch_lo, epoch_hi,
 * 0x414C4732, 0) under key (seed_lo, seed_hi); batch b covers edges [e_s + b*bs, e_s + (b+1)*bs)
 * "while e_e <= |E|".  Writes first_edge[b] (device int64 [cap]) for b < min(nb, cap) and
 * *n_batches = nb (device int64) -- the batch's roots are then (src_i, dst_i, neg_i) of its edges.
 * Errors: TGL_EINVAL unless 0 < chunk_size <= batch_size, n_edges >= 0; TGL_ECAPACITY if
 * cap < n_edges / batch_size.
 */
TGL_API int tgl_chunk_schedule(int64_t n_edges, int64_t batch_size, int64_t chunk_size, uint64_t epoch,
                       uint64_t seed, int64_t *first_edge, int64_t cap, int64_t *n_batches, void *stream);

/* ------------------------------------------------------------------ root staging */

/*
 * The roots of a mini-batch given in TGL's own form -- positive edges (src_i, dst_i, ts_i) and one
 * negative destination neg_i per edge ("600 positive and 600 negative edges") --
 * reading R#16: root 3i = src_i, 3i+1 = dst_i, 3i+2 = neg_i, each at time ts_i.  Writes roots
 * [first_root, first_root + n_roots) of that stream into roots / root_ts (device int32 / float32
 * [n_roots]); the input arrays (device, or mapped pinned host memory) hold the edges
 * first_root / 3 .. (first_root + n_roots - 1) / 3 (index 0 = edge first_root / 3).  Errors:
 * TGL_EINVAL for negative sizes or NULL pointers with n_roots > 0.
 */
TGL_API int tgl_batch_roots(const int32_t *src, const int32_t *dst, const int32_t *neg, const float *ts,
                    int64_t first_root, int64_t n_roots, int32_t *roots, float *root_ts, void *stream);

/* ------------------------------------------------------------------ verification */

/*
 * Per-batch digest of one message-flow block ("a per-batch 64-bit checksum (FNV-1a
 * over offsets, nbr, eid and dt bits)"), so that every batch a timed call produced can be compared
 * with the oracle's output for the same batch without copying the block to the host.  Not a step
 * of Alg. 1: a verification utility.
 * Batch j covers the block's roots [bounds[j], bounds[j+1]) (bounds: device int64 [n_batches+1],
 * non-decreasing, bounds[n_batches] <= the block's n_roots; layer 0: j*B; layer l >= 1: the parent
 * block's offsets at the parent batch bounds).  With e0 = offsets[bounds[j]], e1 =
 * offsets[bounds[j+1]], out[j] (device uint64) is FNV-1a-64 (basis 0xcbf29ce484222325, prime
 * 0x100000001b3) over these bytes, little-endian, in this order:
 *   offsets[i] - e0 as int64 for i = bounds[j] .. bounds[j+1]   (n_j + 1 values, the first 0),
 *   nbr[e0 .. e1), eid[e0 .. e1), then the bit patterns of dt[e0 .. e1)   (32-bit words).
 * One thread per batch (FNV is sequential).  Errors: TGL_EINVAL for n_batches < 0 or a NULL pointer.
 */
TGL_API int tgl_block_digest(const int64_t *offsets, const int32_t *nbr, const int32_t *eid, const float *dt,
                     const int64_t *bounds, int64_t n_batches, uint64_t *out, void *stream);

/* ------------------------------------------------------------------ errors */

/* Synchronises `stream`, returns the first sticky device error raised since the last check by
 * tgl_sample on g (or, when g == NULL, by tgl_gather and tgl_state_write) and clears it. */
TGL_API int tgl_check(tgl_tcsr *g, void *stream);

/* ------------------------------------------------------------------ node-sharded mode */

/*
 * Owner bucketing for the node-sharded T-CSR: node v is owned by shard r with
 * splits[r] <= v < splits[r+1] (splits: device int64 [world+1], splits[0] = 0, splits[world] = V).
 * Stable counting sort of the n roots by owner: perm[j] = index (int32) of the j-th root in
 * (owner, original index) order; counts[r] = roots owned by r (device int64 [world]).  n < 2^31.
 * The exchange itself (all-to-all-v of requests and replies) is NCCL, issued by the caller.
 * workspace >= tgl_shard_bucket_workspace() bytes.
 */
TGL_API int tgl_shard_bucket_workspace(int64_t n_roots, int32_t world, size_t *bytes /* host */);
TGL_API int tgl_shard_bucket(const int32_t *roots, int64_t n_roots, const int64_t *splits, int32_t world,
                     int32_t *perm, int64_t *counts, void *workspace, size_t ws_bytes, void *stream);

/* inv[perm[j]] = j for a permutation perm of [0, n) (device int32): with tgl_gather it returns rows
 * received in bucket order to request order (node-sharded gather of node memory / mailbox rows,
 * SURVEY 8(f) rank 3; the shard-local tables are addressed with global ids through a base pointer
 * offset by -lo rows, valid because owner bucketing only sends a shard ids in [lo, hi)). */
TGL_API int tgl_perm_invert(const int32_t *perm, int64_t n, int32_t *inv, void *stream);

/* counts[i] = offsets[i+1] - offsets[i] (device, int32), e.g. to send a block's per-root counts back. */
TGL_API int tgl_offsets_to_counts(const int64_t *offsets, int64_t n_roots, int32_t *counts, void *stream);

/*
 * Un-permute one reply block: counts_in (int32 per root) / nbr_in / eid_in / dt_in are a CSR block
 * over the roots in BUCKET order (as returned by the owners); the output is the same block in
 * ORIGINAL root order (root perm[j] gets the edges of bucket position j), i.e. exactly what the
 * replicated mode writes.  offsets_out [n+1] int64, edge arrays sized like the inputs.
 */
TGL_API int tgl_shard_unpermute_workspace(int64_t n_roots, size_t *bytes /* host */);
TGL_API int tgl_shard_unpermute(const int32_t *perm, int64_t n_roots, const int32_t *counts_in,
                        const int32_t *nbr_in, const int32_t *eid_in, const float *dt_in,
                        int64_t *offsets_out, int32_t *nbr_out, int32_t *eid_out, float *dt_out,
                        void *workspace, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ node-sharded T-CSR */

/*
 * Build only the lists of the nodes [node_lo, node_hi) of a chronological stream: the rank-local
 * T-CSR of the node-sharded mode (its memory ~ E_s / world).  Same method and bits as
 * tgl_tcsr_build restricted to the logical edges whose owner is in the range: the
 * local lists equal the full build's lists of those nodes, element for element.
 * n_local_stored = the range's E_s (e.g. indptr[node_hi] - indptr[node_lo] of the full degree
 * scan); the call fails with TGL_ECAPACITY if it is not.  Outputs: indptr[node_hi - node_lo + 1]
 * (local, starting at 0), nbr / ts_out / eid_out [n_local_stored] (ts_out 64-byte aligned, padded
 * to a multiple of 16 floats, as tgl_tcsr_build), aux optional (tgl_tcsr_aux_bytes(n_local_stored,
 * node_hi - node_lo)).  The whole stream is validated (synchronously).  The returned handle has its
 * node base set to node_lo (tgl_tcsr_set_node_base): roots and neighbours keep global ids.
 * src / dst / ts / eid may be device memory or mapped pinned host memory (read once per pass).
 */
/* The full graph's indptr [n_nodes+1] only (validation + degree histogram + scan, synchronous like
 * tgl_tcsr_build): what a rank needs to choose edge-balanced node ranges before building its own. */
TGL_API int tgl_tcsr_indptr_workspace(int64_t n_edges, int32_t n_nodes, size_t *bytes /* host */);
TGL_API int tgl_tcsr_indptr(const int32_t *src, const int32_t *dst, const float *ts, int64_t n_edges, int32_t n_nodes,
                    int add_reverse, int64_t *indptr, void *workspace, size_t ws_bytes, void *stream);

TGL_API int tgl_tcsr_build_range_workspace(int64_t n_edges, int32_t n_nodes, int add_reverse, int32_t node_lo,
                                   int32_t node_hi, int64_t n_local_stored, size_t *bytes /* host */);
TGL_API int tgl_tcsr_build_range(const int32_t *src, const int32_t *dst, const float *ts, const int32_t *eid,
                         int64_t n_edges, int32_t n_nodes, int add_reverse, int32_t node_lo, int32_t node_hi,
                         int64_t n_local_stored, int64_t *indptr, int32_t *nbr, float *ts_out, int32_t *eid_out,
                         void *aux, size_t aux_bytes, void *workspace, size_t ws_bytes, void *stream,
                         tgl_tcsr **out /* host */);

/*
 * A rank of the node-sharded sampler: its range's T-CSR handle (node base = splits[rank], e.g.
 * from tgl_tcsr_build_range), the ranges of all ranks (splits: host int64 [world+1], splits[0] = 0,
 * non-decreasing, splits[world] = V) and a transport, exactly one of:
 *   nccl_id  host pointer to TGL_NCCL_ID_BYTES from tgl_shard_nccl_id() on one rank, broadcast to
 *            the others by the caller (e.g. torch.distributed): the library creates an NCCL
 *            communicator of `world` ranks (one process per GPU, the current device);
 *   group    an in-process group (tgl_shard_group_create): ranks are threads of one process that
 *            exchange by device copies -- for tests and single-device runs.
 * Ownership: the shard borrows `local` (it must outlive the shard) and owns its communicator and
 * its internal device buffers (grown by tgl_sample_sharded on first use, freed by
 * tgl_shard_destroy).  Errors: TGL_EINVAL (bad splits, local range != splits[rank]..splits[rank+1],
 * both or neither transport), TGL_ENCCL (NCCL missing or communicator creation failed).
 */
#define TGL_NCCL_ID_BYTES 128
typedef struct tgl_shard tgl_shard;             /* opaque, host-side */
typedef struct tgl_shard_group tgl_shard_group; /* opaque, host-side */
TGL_API int tgl_shard_nccl_id(void *id /* host, TGL_NCCL_ID_BYTES */);
TGL_API int tgl_shard_group_create(int32_t world, tgl_shard_group **out /* host */);
TGL_API int tgl_shard_group_destroy(tgl_shard_group *group);
TGL_API int tgl_shard_create(const tgl_tcsr *local, const int64_t *splits /* host [world+1] */, int32_t rank,
                     int32_t world, const void *nccl_id /* host or NULL */, tgl_shard_group *group /* or NULL */,
                     tgl_shard **out /* host */);
TGL_API int tgl_shard_destroy(tgl_shard *shard);

/*
 * tgl_sample over a node-sharded T-CSR: a COLLECTIVE call -- every rank of the shard's group calls
 * it (with its own roots, possibly none) with the same n_layers / fanouts / strategy / snapshots /
 * seed.  The caller's blocks (capacities from tgl_sample_capacity, as for tgl_sample) receive
 * exactly the bits tgl_sample writes on the full T-CSR for these roots with this root_key_base
 * (R#7 keys travel with the requests, R#3 lower bounds too).  Per chain (layer 0 with its S blocks,
 * then one per (layer, snapshot)): owner bucketing, an all-to-all of counts, the requests, local
 * sampling on the owner's range, an all-to-all of reply sizes and the replies (grouped NCCL
 * send / recv), un-permute -- two host synchronisations per chain (the sizes of the variable
 * exchanges).  Stream-ordered on `stream`; the blocks' n_roots_dev / nnz_dev are written on the
 * device.  Options of tgl_sample_ex (dedup, validity, hop-root time) are not supported here.
 */
TGL_API int tgl_sample_sharded(tgl_shard *shard, const int32_t *roots, const float *root_ts, int64_t n_roots,
                       int32_t n_layers, const int32_t *fanouts /* host [L] */, tgl_strategy strategy,
                       int32_t n_snapshots, float snapshot_len, uint64_t seed, uint64_t root_key_base,
                       tgl_block *out /* host [L*S] */, void *stream);

/*
 * Sharded node state: node memory / mailbox tables split
 * by the shard's node ranges -- rank r holds the rows of global nodes [splits[r], splits[r+1]).
 * COLLECTIVE calls (every rank of the shard calls them, with its own ids, possibly none).
 *
 * tgl_shard_gather (Fig. 2 step 2 across ranks): for every table j, out_j[i] = the row of global
 *   node ids[i] (wherever it lives), i < n, in request order.  tables[j].table = this rank's LOCAL
 *   rows, tables[j].n_rows = splits[rank+1] - splits[rank], tables[j].row_bytes = bytes per node
 *   (a K-slot ring is one K * slot-bytes row), tables[j].out = device [n * row_bytes].
 *   id == -1 gives a zero row.  One host synchronisation (the request counts).
 * tgl_shard_state_write (Fig. 2 step 6 across ranks, R#25): the events (ids[i], ts[i], rows_j[i])
 *   of all ranks are applied, in (rank, event index) order, to the owners' LOCAL tables exactly as
 *   tgl_state_write applies a batch (ts: device float [n], required when n > 0, the same fields
 *   travel from every rank): tables[j].rows = device [n * row_bytes], tables[j].table =
 *   LOCAL [n_local * K * row_bytes]; pos (int32 [n_local], required for K > 1) and ts_table
 *   (float [n_local * K], may be NULL) are LOCAL too.  At most TGL_MAX_GATHER_TABLES - 2 tables.
 *   One host synchronisation.  Device-detected errors go to tgl_check(NULL, ...).
 */
TGL_API int tgl_shard_gather(tgl_shard *shard, const int32_t *ids, int64_t n,
                     const tgl_gather_table *tables /* host [n_tables] */, int32_t n_tables, void *stream);
TGL_API int tgl_shard_state_write(tgl_shard *shard, const int32_t *ids, const float *ts, int64_t n, int32_t K,
                          int32_t *pos, float *ts_table, const tgl_state_table *tables /* host [n_tables] */,
                          int32_t n_tables, void *stream);

/* Cumulative exchange statistics of a shard: bytes sent to / received from OTHER ranks (the
 * NVLink traffic of the protocol) and host synchronisations. */
TGL_API int tgl_shard_stats(const tgl_shard *shard, int64_t *bytes_sent, int64_t *bytes_recv,
                    int64_t *host_syncs);

#ifdef __cplusplus
}
#endif
#endif /* TGL_H_ */
