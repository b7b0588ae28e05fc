"""ctypes declarations of libtgl.so (include/tgl.h).  Argument marshalling only.

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``) next to this
file.  There is no fallback: if it is missing or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TGL_LIB_PATH") or os.path.join(_HERE, "libtgl.so")  # override: experiments only

OK, EINVAL, ERANGE, EUNSORTED, ECAPACITY, EWORKSPACE, ECUDA, ENCCL, ENOTSUP = 0, -1, -2, -3, -4, -5, -6, -7, -8
MOST_RECENT, UNIFORM = 0, 1
MAX_SNAPSHOTS, MAX_FANOUT, MAX_GATHER_TABLES = 16, 1024, 8
NCCL_ID_BYTES = 128

P = ctypes.c_void_p
i32, i64, u64, f32, sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_size_t


class Block(ctypes.Structure):
    """tgl_block (include/tgl.h)."""
    _fields_ = [("cap_roots", i64), ("cap_edges", i64), ("offsets", P), ("nbr", P), ("eid", P), ("dt", P),
                ("ts_edge", P), ("n_roots_dev", P), ("nnz_dev", P)]


MAX_FUSED_GATHER = 8


class FusedTable(ctypes.Structure):
    """tgl_fused_table (include/tgl.h)."""
    _fields_ = [("table", P), ("n_rows", i64), ("row_bytes", i64), ("out", P), ("by_edge", i32)]


class FusedGather(ctypes.Structure):
    """tgl_fused_gather (include/tgl.h)."""
    _fields_ = [("n_tables", i32), ("tables", FusedTable * MAX_FUSED_GATHER)]


class SampleOptions(ctypes.Structure):
    _fields_ = [("hop_time", ctypes.c_int32), ("replacement", ctypes.c_int32), ("dedup", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 5), ("edge_valid", ctypes.c_void_p),
                ("gather", ctypes.POINTER(FusedGather))]


class DedupBlock(ctypes.Structure):
    """tgl_dedup_block (include/tgl.h)."""
    _fields_ = [("cap", i64), ("src_index", P), ("uniq_node", P), ("uniq_ts", P), ("n_uniq_dev", P)]


class StateTable(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_void_p), ("row_bytes", ctypes.c_int64), ("table", ctypes.c_void_p)]


class GatherTable(ctypes.Structure):
    """tgl_gather_table (include/tgl.h)."""
    _fields_ = [("table", P), ("n_rows", i64), ("row_bytes", i64), ("out", P)]


# name -> (restype, argtypes), exactly the declarations of include/tgl.h
SIGNATURES = {
    "tgl_abi_version": (ctypes.c_int, []),
    "tgl_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "tgl_tcsr_build_workspace": (ctypes.c_int, [i64, i32, ctypes.c_int, ctypes.POINTER(sz)]),
    "tgl_tcsr_build": (ctypes.c_int, [P, P, P, P, i64, i32, ctypes.c_int, P, P, P, P, P, sz, P, sz, P,
                                      ctypes.POINTER(P)]),
    "tgl_tcsr_aux_bytes": (ctypes.c_int, [i64, i32, ctypes.POINTER(sz)]),
    "tgl_tcsr_aux_build": (ctypes.c_int, [P, P, P, P, i32, i64, P, sz, P]),
    "tgl_tcsr_wrap": (ctypes.c_int, [P, P, P, P, P, sz, i32, i64, ctypes.POINTER(P)]),
    "tgl_tcsr_destroy": (ctypes.c_int, [P]),
    "tgl_tcsr_info": (ctypes.c_int, [P, ctypes.POINTER(i32), ctypes.POINTER(i64)]),
    "tgl_tcsr_codec": (ctypes.c_int, [P, ctypes.POINTER(i32), ctypes.POINTER(i32)]),
    "tgl_sample_capacity": (ctypes.c_int, [i64, i32, P, i32, ctypes.c_int, f32, P, P, ctypes.POINTER(sz)]),
    "tgl_sample": (ctypes.c_int, [P, P, P, i64, i32, P, ctypes.c_int, i32, f32, u64, u64, P, P, sz, P]),
    "tgl_sample_keyed": (ctypes.c_int, [P, P, P, P, i64, i32, P, ctypes.c_int, i32, f32, u64, P, P, sz, P]),
    "tgl_sample_ex": (ctypes.c_int, [P, P, P, P, i64, i32, P, ctypes.c_int, i32, f32, u64, u64, P, P, P, P, sz, P]),
    "tgl_sample_capacity_ex": (ctypes.c_int, [i64, i32, P, i32, ctypes.c_int, f32, P, P, P, ctypes.POINTER(sz)]),
    "tgl_tcsr_set_node_base": (ctypes.c_int, [P, i64]),
    "tgl_shard_unpermute_workspace": (ctypes.c_int, [i64, ctypes.POINTER(sz)]),
    "tgl_offsets_to_counts": (ctypes.c_int, [P, i64, P, P]),
    "tgl_shard_unpermute": (ctypes.c_int, [P, i64, P, P, P, P, P, P, P, P, P, sz, P]),
    "tgl_gather": (ctypes.c_int, [P, i64, P, P, i32, P]),
    "tgl_chunk_schedule": (ctypes.c_int, [i64, i64, i64, u64, u64, P, i64, P, P]),
    "tgl_edge_valid_set": (ctypes.c_int, [P, i64, P, i64, i32, P]),
    "tgl_perm_invert": (ctypes.c_int, [P, i64, P, P]),
    "tgl_state_write_workspace": (ctypes.c_int, [i64, i32, ctypes.POINTER(sz)]),
    "tgl_state_write": (ctypes.c_int, [P, P, i64, i32, i32, P, P, P, i32, P, sz, P]),
    "tgl_check": (ctypes.c_int, [P, P]),
    "tgl_block_digest": (ctypes.c_int, [P, P, P, P, P, i64, P, P]),
    "tgl_batch_roots": (ctypes.c_int, [P, P, P, P, i64, i64, P, P, P]),
    "tgl_tcsr_indptr_workspace": (ctypes.c_int, [i64, i32, ctypes.POINTER(sz)]),
    "tgl_tcsr_indptr": (ctypes.c_int, [P, P, P, i64, i32, ctypes.c_int, P, P, sz, P]),
    "tgl_tcsr_build_range_workspace": (ctypes.c_int, [i64, i32, ctypes.c_int, i32, i32, i64, ctypes.POINTER(sz)]),
    "tgl_tcsr_build_range": (ctypes.c_int, [P, P, P, P, i64, i32, ctypes.c_int, i32, i32, i64, P, P, P, P, P, sz, P,
                                            sz, P, ctypes.POINTER(P)]),
    "tgl_shard_nccl_id": (ctypes.c_int, [P]),
    "tgl_shard_group_create": (ctypes.c_int, [i32, ctypes.POINTER(P)]),
    "tgl_shard_group_destroy": (ctypes.c_int, [P]),
    "tgl_shard_create": (ctypes.c_int, [P, P, i32, i32, P, P, ctypes.POINTER(P)]),
    "tgl_shard_destroy": (ctypes.c_int, [P]),
    "tgl_sample_sharded": (ctypes.c_int, [P, P, P, i64, i32, P, ctypes.c_int, i32, f32, u64, u64, P, P]),
    "tgl_shard_gather": (ctypes.c_int, [P, P, i64, P, i32, P]),
    "tgl_shard_state_write": (ctypes.c_int, [P, P, P, i64, i32, P, P, P, i32, P]),
    "tgl_shard_stats": (ctypes.c_int, [P, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)]),
    "tgl_shard_bucket_workspace": (ctypes.c_int, [i64, i32, ctypes.POINTER(sz)]),
    "tgl_shard_bucket": (ctypes.c_int, [P, i64, P, i32, P, P, P, sz, P]),
}


def load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libtgl.so not built at {LIB_PATH}: run `make` or __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class TGLError(RuntimeError):
    def __init__(self, code: int, what: str, lib=None):
        msg = lib.tgl_strerror(code).decode() if lib is not None else str(code)
        super().__init__(f"{what}: {msg} ({code})")
        self.code = code
