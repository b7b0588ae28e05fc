"""CPU parity oracle for the TGL hot path (arXiv 2203.14883) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_2203_14883_b200``) never imports it, and it never imports the product path:
the two share no code.  The arithmetic lives in ``tgl_oracle.c`` (plain C, one thread,
``-ffp-contract=off``); this module only marshals numpy arrays through ctypes and
composes Alg. 1's layer/snapshot loop out of single blocks.

``oracle/brute.py`` is the second, independent level of the test pyramid: a numpy
brute force over the whole logical edge stream (no T-CSR, no binary search).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import Iterable, List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tgl_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, ERANGE, EUNSORTED = 0, -1, -2, -3
MOST_RECENT, UNIFORM = 0, 1

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
          "-fexcess-precision=standard", "-fPIC", "-shared"]


def compile_lib(force: bool = False) -> str:
    """Compile tgl_oracle.c into oracle/liboracle.so (gcc, plain C)."""
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(compile_lib())
        P = ctypes.c_void_p
        i64, i32, f32, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_float, ctypes.c_uint64
        L.oracle_philox4x32_10.argtypes = [P, P, P]
        L.oracle_philox4x32_10.restype = None
        L.oracle_tcsr_build.argtypes = [P, P, P, P, i64, i32, ctypes.c_int, P, P, P, P, P]
        L.oracle_tcsr_build.restype = ctypes.c_int
        L.oracle_tcsr_count.argtypes = [P, P, P, i64, i32, ctypes.c_int, P, f32, ctypes.c_int, P]
        L.oracle_tcsr_count.restype = ctypes.c_int
        L.oracle_tcsr_fill.argtypes = [P, P, P, P, i64, i64, i32, ctypes.c_int, P, P, P, P, P]
        L.oracle_tcsr_fill.restype = ctypes.c_int
        L.oracle_sample_block.argtypes = [P, P, P, P, i32, P, P, P, P, i64, i32, i32, f32, i32, i32,
                                          i32, u64, P, P, P, P, P, P, P, P, P, P, P]
        L.oracle_sample_block.restype = i64
        L.oracle_gather.argtypes = [P, i64, P, i64, i64, P, P]
        L.oracle_gather.restype = None
        L.oracle_state_write.argtypes = [P, P, i64, i32, i32, P, P, P, i64, P, P]
        L.oracle_state_write.restype = None
        L.oracle_fnv1a64.argtypes = [P, i64, u64]
        L.oracle_fnv1a64.restype = u64
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle error {code}")
        self.code = code


# --------------------------------------------------------------------------- Philox
def philox4x32_10(ctr, key) -> np.ndarray:
    """Philox4x32-10 block (Salmon et al. SC'11): ctr = 4 x u32, key = 2 x u32."""
    c = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32))
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32))
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


# --------------------------------------------------------------------------- T-CSR
class TCSR(dict):
    """indptr int64 [V+1]; nbr int32, ts float32, eid int32 [E_s]."""

    @property
    def n_nodes(self) -> int:
        return len(self["indptr"]) - 1


def build(src, dst, ts, eid=None, *, n_nodes: int, add_reverse: bool) -> TCSR:
    """Counting-sort T-CSR of the logical edge stream (R#19)."""
    src = np.ascontiguousarray(src, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    ts = np.ascontiguousarray(ts, dtype=np.float32)
    eid = None if eid is None else np.ascontiguousarray(eid, dtype=np.int32)
    E = len(src)
    Es = E * (2 if add_reverse else 1)
    indptr = np.zeros(n_nodes + 1, dtype=np.int64)
    nbr = np.zeros(Es, dtype=np.int32)
    ts_out = np.zeros(Es, dtype=np.float32)
    eid_out = np.zeros(Es, dtype=np.int32)
    cursor = np.zeros(max(n_nodes, 1), dtype=np.int64)
    rc = lib().oracle_tcsr_build(_p(src), _p(dst), _p(ts), _p(eid), E, n_nodes, int(add_reverse),
                                 _p(indptr), _p(nbr), _p(ts_out), _p(eid_out), _p(cursor))
    if rc != OK:
        raise OracleError(rc, "tcsr_build")
    return TCSR(indptr=indptr, nbr=nbr, ts=ts_out, eid=eid_out)


def build_restricted(chunks: Iterable, *, n_nodes: int, add_reverse: bool,
                     keep: np.ndarray) -> TCSR:
    """T-CSR restricted to owners with keep[v] (same counting sort, two streaming passes).

    ``chunks`` is a zero-argument callable returning an iterator of
    (src, dst, ts, eid_or_None, eid_base) numpy chunks in stream order; it is called
    twice (count pass, fill pass).  Lists of kept nodes are identical to the full
    build's; other nodes get empty lists.  Used where the full host T-CSR is not needed
    (billion-edge configs, where only the sampled roots' lists are read).
    """
    keep = np.ascontiguousarray(keep, dtype=np.uint8)
    deg = np.zeros(n_nodes, dtype=np.int64)
    prev, have_prev = 0.0, 0
    for (s, d, t, e, base) in chunks():
        s = np.ascontiguousarray(s, dtype=np.int32)
        d = np.ascontiguousarray(d, dtype=np.int32)
        t = np.ascontiguousarray(t, dtype=np.float32)
        rc = lib().oracle_tcsr_count(_p(s), _p(d), _p(t), len(s), n_nodes, int(add_reverse), _p(keep),
                                     float(prev), have_prev, _p(deg))
        if rc != OK:
            raise OracleError(rc, "tcsr_count")
        if len(t):
            prev, have_prev = float(t[-1]), 1
    indptr = np.zeros(n_nodes + 1, dtype=np.int64)
    np.cumsum(deg, out=indptr[1:])
    Es = int(indptr[-1])
    nbr = np.zeros(Es, dtype=np.int32)
    ts_out = np.zeros(Es, dtype=np.float32)
    eid_out = np.zeros(Es, dtype=np.int32)
    cursor = indptr[:-1].copy()
    for (s, d, t, e, base) in chunks():
        s = np.ascontiguousarray(s, dtype=np.int32)
        d = np.ascontiguousarray(d, dtype=np.int32)
        t = np.ascontiguousarray(t, dtype=np.float32)
        e = None if e is None else np.ascontiguousarray(e, dtype=np.int32)
        rc = lib().oracle_tcsr_fill(_p(s), _p(d), _p(t), _p(e), int(base), len(s), n_nodes,
                                    int(add_reverse), _p(keep), _p(cursor), _p(nbr), _p(ts_out),
                                    _p(eid_out))
        if rc != OK:
            raise OracleError(rc, "tcsr_fill")
    return TCSR(indptr=indptr, nbr=nbr, ts=ts_out, eid=eid_out)


# --------------------------------------------------------------------------- sampler
def sample_block(g: TCSR, root_node, root_ts, root_key, root_lo, *, layer: int, snapshot: int,
                 snapshot_len: float, k: int, strategy: int, seed: int,
                 want_children: bool, replacement: bool = False, edge_valid=None) -> dict:
    """One (layer, snapshot) block of Alg. 1 -- see tgl_oracle.c."""
    root_node = np.ascontiguousarray(root_node, dtype=np.int32)
    root_ts = np.ascontiguousarray(root_ts, dtype=np.float32)
    root_key = np.ascontiguousarray(root_key, dtype=np.uint64)
    root_lo = None if root_lo is None else np.ascontiguousarray(root_lo, dtype=np.float32)
    n = len(root_node)
    cap = n * k
    offsets = np.zeros(n + 1, dtype=np.int64)
    nbr = np.zeros(cap, dtype=np.int32)
    eid = np.zeros(cap, dtype=np.int32)
    dt = np.zeros(cap, dtype=np.float32)
    ts_edge = np.zeros(cap, dtype=np.float32) if want_children else None
    ckey = np.zeros(cap, dtype=np.uint64) if want_children else None
    clo = np.zeros(cap, dtype=np.float32) if want_children else None
    err = np.zeros(1, dtype=np.int32)
    scratch = np.zeros(max(k, 1), dtype=np.uint32)
    cand = None
    if edge_valid is not None:
        edge_valid = np.ascontiguousarray(edge_valid, dtype=np.uint32)
        cand = np.zeros(max(int(np.max(np.diff(g["indptr"]), initial=0)), 1), dtype=np.int64)
    nnz = lib().oracle_sample_block(_p(g["indptr"]), _p(g["nbr"]), _p(g["ts"]), _p(g["eid"]),
                                    g.n_nodes, _p(root_node), _p(root_ts), _p(root_key), _p(root_lo), n,
                                    layer, snapshot, float(snapshot_len), k, strategy, int(bool(replacement)),
                                    int(seed) & 0xFFFFFFFFFFFFFFFF, _p(offsets), _p(nbr), _p(eid), _p(dt),
                                    _p(ts_edge), _p(ckey), _p(clo), _p(err), _p(scratch), _p(edge_valid), _p(cand))
    out = dict(offsets=offsets, nbr=nbr[:nnz], eid=eid[:nnz], dt=dt[:nnz], err=int(err[0]))
    if want_children:
        out.update(ts_edge=ts_edge[:nnz], child_key=ckey[:nnz], child_lo=clo[:nnz])
    return out


def sample(g: TCSR, roots, root_ts, *, fanouts: List[int], strategy: int, n_snapshots: int = 1,
           snapshot_len: float = math.inf, seed: int = 0, root_key_base: int = 0,
           hop_time: str = "edge", replacement: bool = False, dedup: bool = False,
           edge_valid=None) -> List[dict]:
    """Alg. 1: L x S blocks, block (l, s) at index l*S + s.

    Layer-0 roots are the caller's; the roots of block (l, s), l >= 1, are the outputs
    (nbr, ts_edge) of block (l-1, s) in output order, without dedup (R#14), each with
    root key parent_key * k_{l-1} + j (R#7) and inherited lower bound (R#3).
    Variants: hop_time="root" -- hop roots carry their parent's root time
    instead of the sampled edge's ("others use the root's timestamp", R#23);
    replacement=True -- uniform draws with replacement (R#24).
    dedup=True (R#27, SPEC's MFG): every block also lists the distinct (node, hop time) pairs of its
    outputs in order of first appearance (uniq_node, uniq_ts, bit-exact equality of the time) with
    src_index[i] = the pair of output i; the next layer's roots are that list, each keyed by its
    first occurrence's child key.  Not defined with inherited finite lower bounds (L > 1 with a
    finite snapshot length): different windows would merge.
    edge_valid (uint32 bitmask over edge ids, R#28, P:L258 / L556): invalid edges are not candidates.
    """
    if hop_time not in ("edge", "root"):
        raise ValueError("hop_time must be 'edge' or 'root'")
    L, S = len(fanouts), int(n_snapshots)
    if dedup and L > 1 and math.isfinite(snapshot_len):
        raise ValueError("dedup needs S == 1 or an infinite snapshot length when L > 1 (R#27)")
    root_node = np.ascontiguousarray(np.asarray(roots, dtype=np.int32))
    root_ts = np.ascontiguousarray(np.asarray(root_ts, dtype=np.float32))
    n = len(root_node)
    keys0 = (np.uint64(root_key_base) + np.arange(n, dtype=np.uint64)).astype(np.uint64)
    need_lo = L > 1 and math.isfinite(snapshot_len)
    blocks: List[Optional[dict]] = [None] * (L * S)
    for s in range(S):
        rn, rt, rk, rlo = root_node, root_ts, keys0, None
        for l in range(L):
            want = l < L - 1
            b = sample_block(g, rn, rt, rk, rlo, layer=l, snapshot=s, snapshot_len=snapshot_len,
                             k=fanouts[l], strategy=strategy, seed=seed, want_children=want or dedup,
                             replacement=replacement, edge_valid=edge_valid)
            if want or dedup:
                # R#4 / R#23: the hop root's time is the sampled edge's, or its parent root's
                t_next = b["ts_edge"] if hop_time == "edge" else np.repeat(rt, np.diff(b["offsets"]))
                t_next = np.ascontiguousarray(t_next, dtype=np.float32)
            if dedup:
                first, src_index = {}, np.zeros(len(b["nbr"]), dtype=np.int32)
                order = []
                for i, (v, tb) in enumerate(zip(b["nbr"].tolist(), t_next.view(np.uint32).tolist())):
                    if (v, tb) not in first:
                        first[(v, tb)] = len(order)
                        order.append(i)
                    src_index[i] = first[(v, tb)]
                order = np.array(order, dtype=np.int64)
                b["src_index"], b["uniq_node"], b["uniq_ts"] = src_index, b["nbr"][order], t_next[order]
                b["uniq_key"] = b["child_key"][order]
                if not want:
                    for key in ("ts_edge", "child_key", "child_lo"):
                        b.pop(key, None)
            blocks[l * S + s] = b
            if want:
                if dedup:
                    rn, rt, rk = b["uniq_node"], b["uniq_ts"], b["uniq_key"]
                else:
                    rn, rt, rk = b["nbr"], t_next, b["child_key"]
                rlo = b["child_lo"] if need_lo else None
    return blocks


# --------------------------------------------------------------------------- gather
def gather(ids, table: np.ndarray) -> (np.ndarray, int):
    """out[i] = table[ids[i]] byte for byte; id -1 -> zero row (Fig. 2 step 2)."""
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    table = np.ascontiguousarray(table)
    n_rows = table.shape[0]
    row_bytes = table.nbytes // max(n_rows, 1) if n_rows else int(np.prod(table.shape[1:])) * table.itemsize
    out = np.zeros((len(ids),) + table.shape[1:], dtype=table.dtype)
    err = np.zeros(1, dtype=np.int32)
    lib().oracle_gather(_p(ids), len(ids), _p(table), n_rows, row_bytes, _p(out), _p(err))
    return out, int(err[0])


# --------------------------------------------------------------------------- state write
def state_write(ids, ts, *, n_nodes: int, K: int, tables, pos=None, ts_table=None) -> int:
    """Fig. 2 step 6, reading R#25: events applied in batch order, each into
    slot pos[v] of node v's K-slot ring, pos[v] = (pos[v] + 1) mod K.  tables: list of
    (rows [n, ...], table [n_nodes * K, ...]) numpy pairs, updated IN PLACE; pos (int32 [n_nodes])
    and ts_table (float32 [n_nodes * K]) likewise.  Returns the error code (0 or ERANGE)."""
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    ts = np.ascontiguousarray(ts, dtype=np.float32)
    n = len(ids)
    err = np.zeros(1, dtype=np.int32)
    pos_start = None if pos is None else pos.copy()
    jobs = list(tables) if tables else [(None, None)]
    last = None
    for j, (rows, table) in enumerate(jobs):
        p = None if pos is None else pos_start.copy()  # every table sees the same ring cursors
        rb = 0
        if rows is not None:
            assert rows.flags.c_contiguous and table.flags.c_contiguous
            rb = rows.nbytes // n if n else 0
        lib().oracle_state_write(_p(ids), _p(ts), n, n_nodes, K, _p(p), _p(ts_table if j == 0 else None),
                                 _p(rows), rb, _p(table), _p(err))
        last = p
    if pos is not None:
        pos[:] = last
    return int(err[0])


# --------------------------------------------------------------------------- Alg. 2
def chunk_schedule(n_edges: int, bs: int, cs: int, epoch: int, seed: int) -> List[int]:
    """Random chunk scheduling, Alg. 2, reading R#26: per epoch the first batch
    starts at e_s = r * cs, r uniform in [0, bs // cs) (Philox word 0, counter (epoch_lo, epoch_hi,
    0x414C4732, 0), key = seed); batches are [e_s + b*bs, e_s + (b+1)*bs) while the end <= |E|.
    Returns the first edge of every batch of the epoch, in order."""
    if bs <= 0 or cs <= 0 or cs > bs or n_edges < 0 or epoch < 0:
        raise ValueError("need 0 < cs <= bs, n_edges >= 0, epoch >= 0")
    ctr = np.array([epoch & 0xFFFFFFFF, (epoch >> 32) & 0xFFFFFFFF, 0x414C4732, 0], dtype=np.uint32)
    key = np.array([seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF], dtype=np.uint32)
    x = int(philox4x32_10(ctr, key)[0])
    r = (x * (bs // cs)) >> 32
    e_s, out = r * cs, []
    while e_s + bs <= n_edges:          # "while e_e <= |E|"
        out.append(e_s)
        e_s += bs
    return out


# --------------------------------------------------------------------------- checksums (test infra)
FNV_BASIS = 0xcbf29ce484222325


def fnv1a64(data: bytes | np.ndarray, h: int = FNV_BASIS) -> int:
    """64-bit FNV-1a over the bytes of `data`, continuing from h (tgl_oracle.c)."""
    a = np.ascontiguousarray(np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray))
                             else np.asarray(data).view(np.uint8).reshape(-1))
    return int(lib().oracle_fnv1a64(_p(a), a.size, h))


def block_digest(block: dict) -> int:
    """Digest of one oracle block in the byte order of tgl_block_digest (include/tgl.h): offsets
    rebased to the block's first root (int64), then nbr, eid and the dt bit patterns."""
    off = np.ascontiguousarray(block["offsets"] - block["offsets"][0], dtype="<i8")
    h = fnv1a64(off)
    h = fnv1a64(np.ascontiguousarray(block["nbr"], dtype="<i4"), h)
    h = fnv1a64(np.ascontiguousarray(block["eid"], dtype="<i4"), h)
    return fnv1a64(np.ascontiguousarray(block["dt"], dtype="<f4").view("<u4"), h)
