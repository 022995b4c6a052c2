"""ctypes view of include/csattn_b200.h (the C ABI of libcsattn_b200.so).

The shared library is built in-tree by __graft_entry__.build() (make -C
paper_2604_08584_b200/csrc). Loading fails loudly when it is missing: there is
no Python or CPU fallback for any compute entry point.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcsattn_b200.so")

HOST_BUFFERS = 0x1
NO_SYNC = 0x2

STATUS_NAMES = {
    0: "ok", 1: "Error", 2: "DimensionError", 3: "ParameterError", 4: "DataError",
    5: "BadMagicError", 6: "VersionError", 7: "TruncatedError", 8: "CorruptError",
    9: "PropertyError", 10: "StreamExhaustedError", 20: "CudaError", 21: "CapacityError",
}


class PrefillRowsC(C.Structure):
    _fields_ = [("queries", C.c_void_p), ("n_queries", C.c_uint64), ("keys", C.c_void_p),
                ("values", C.c_void_p), ("n_rows", C.c_uint64)]


class IndexConfigC(C.Structure):
    _fields_ = [("alpha", C.c_double), ("list_capacity", C.c_uint64),
                ("normalize_keys", C.c_int32), ("score_bits", C.c_int32),
                ("centroids", C.c_uint64), ("iterations", C.c_uint64),
                ("batch_size", C.c_uint64), ("seed", C.c_uint64), ("tolerance", C.c_double)]


class RetrievalConfigC(C.Structure):
    _fields_ = [("keep_ratio", C.c_double), ("search_period", C.c_uint64),
                ("recent_window", C.c_uint64), ("weights", C.POINTER(C.c_double)),
                ("n_weights", C.c_uint64), ("backoff_tau", C.c_uint64),
                ("backoff_threshold", C.c_double), ("recent_passthrough", C.c_int32),
                ("reserved", C.c_int32)]


class SyntheticSpecC(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("dim", C.c_uint64), ("clusters", C.c_uint64),
                ("seed", C.c_uint64), ("plant_fraction", C.c_double),
                ("plant_scale", C.c_double), ("query_noise", C.c_double), ("dwell", C.c_uint64)]


class StepReportC(C.Structure):
    _fields_ = [("k", C.c_uint64), ("searched", C.c_int32), ("reserved", C.c_int32),
                ("centroid_dot_ops", C.c_uint64), ("gathered_entries", C.c_uint64),
                ("reduce_ops", C.c_uint64), ("attention_key_ops", C.c_uint64),
                ("h2d_bytes_model", C.c_double), ("searches", C.c_uint64),
                ("inserts_attempted", C.c_uint64), ("inserts_applied", C.c_uint64),
                ("insert_dot_ops", C.c_uint64), ("worst_best_cosine", C.c_double)]


class SessionInfoC(C.Structure):
    _fields_ = [("dim", C.c_uint64), ("subspaces", C.c_uint64), ("centroids", C.c_uint64),
                ("list_capacity", C.c_uint64), ("prefill_len", C.c_uint64),
                ("context_len", C.c_uint64), ("steps", C.c_uint64), ("max_context", C.c_uint64),
                ("group", C.c_uint64), ("alpha", C.c_double), ("normalize_keys", C.c_int32),
                ("score_bits", C.c_int32), ("device_bytes", C.c_uint64)]


vp = C.c_void_p
u64 = C.c_uint64
u32 = C.c_uint32
i32 = C.c_int32
P = C.POINTER

# name -> (restype, argtypes); every symbol include/csattn_b200.h declares
class ShardIoC(C.Structure):
    _fields_ = [("q", C.c_void_p), ("new_keys", C.c_void_p), ("new_values", C.c_void_p),
                ("ghist", C.c_void_p), ("bucket", C.c_void_p), ("bucket_all", C.c_void_p),
                ("counts", C.c_void_p), ("counts_all", C.c_void_p),
                ("partial", C.c_void_p), ("partial_all", C.c_void_p), ("out", C.c_void_p),
                ("selected", C.c_void_p), ("n_selected", C.c_void_p), ("sel_stride", C.c_uint64),
                ("victim", C.c_void_p), ("spec_fail", C.c_void_p), ("shard_index", C.c_uint32),
                ("n_shards", C.c_uint32)]


SHARD_SCAN, SHARD_BUCKET, SHARD_MARK, SHARD_EMIT, SHARD_MERGE, SHARD_VICTIM, SHARD_INSERT, \
    SHARD_RESCAN = range(8)

CSAT_MAX_SUBSPACES = 32


class CsatHeaderC(C.Structure):
    _fields_ = [("m", C.c_uint64), ("centroids", C.c_uint64), ("list_capacity", C.c_uint64),
                ("dim", C.c_uint64), ("prefill_len", C.c_uint64), ("score_bits", C.c_int32),
                ("normalize_keys", C.c_int32), ("widths", C.c_uint64 * CSAT_MAX_SUBSPACES)]


SIGNATURES = {
    "csattn_index_config_default": (None, [P(IndexConfigC)]),
    "csattn_retrieval_config_default": (None, [P(RetrievalConfigC)]),
    "csattn_synthetic_spec_default": (None, [P(SyntheticSpecC)]),
    "csattn_keep_count": (C.c_int, [C.c_double, u64, P(u64)]),
    "csattn_parse_schedule": (C.c_int, [C.c_char_p, P(C.c_double), P(u64)]),
    "csattn_h2d_bytes": (C.c_int, [C.c_double, u64, u64, u64, u64, P(C.c_double)]),
    "csattn_make_synthetic": (C.c_int, [P(SyntheticSpecC), vp, vp, vp]),
    "csattn_last_error": (C.c_char_p, []),
    "csattn_status_name": (C.c_char_p, [C.c_int]),
    "csattn_ctx_create": (C.c_int, [C.c_int, vp, P(vp)]),
    "csattn_ctx_destroy": (C.c_int, [vp]),
    "csattn_ctx_synchronize": (C.c_int, [vp]),
    "csattn_ctx_launch_count": (u64, [vp]),
    "csattn_ctx_build_stats": (C.c_int, [vp, P(u64), P(u64)]),
    "csattn_ctx_profile": (C.c_int, [vp, i32]),
    "csattn_ctx_profile_read": (C.c_int, [vp, P(C.c_double), P(u64), i32]),
    "csattn_prefill": (C.c_int, [vp, vp, u64, vp, vp, u64, u64, P(u64), u64, P(IndexConfigC),
                                 P(RetrievalConfigC), u64, u64, u32, P(vp)]),
    "csattn_prefill_batch": (C.c_int, [vp, u64, P(PrefillRowsC), u64, P(u64), u64, P(IndexConfigC),
                                       P(RetrievalConfigC), u64, u64, u32, P(vp)]),
    "csattn_prefill_from_centroids": (C.c_int, [vp, vp, u64, vp, vp, u64, u64, P(u64), u64,
                                                P(IndexConfigC), P(RetrievalConfigC), u64, u64,
                                                u32, P(vp)]),
    "csattn_session_import": (C.c_int, [vp, vp, u64, vp, vp, vp, u64, u64, C.c_double, i32, i32,
                                        vp, vp, u64, u64, P(u64), u64, P(RetrievalConfigC), u64,
                                        u64, P(vp)]),
    "csattn_session_export": (C.c_int, [vp, vp, vp, vp, u64, vp]),
    "csattn_session_centroids": (C.c_int, [vp, vp]),
    "csattn_shard_create": (C.c_int, [vp, vp, u64, u64, C.c_int32, u64, P(vp)]),
    "csattn_shard_buffer_words": (C.c_int, [vp, P(u64), P(u64), P(u64), P(u64)]),
    "csattn_shard_step": (C.c_int, [vp, u64, P(vp), C.c_int32, P(ShardIoC)]),
    "csattn_dense_topk": (C.c_int, [vp, vp, u64, vp, u32]),
    "csattn_ctx_stream": (vp, [vp]),
    "csattn_buffer_add_u32": (C.c_int, [vp, vp, vp, u64]),
    "csattn_buffer_min_u64": (C.c_int, [vp, vp, vp, u64]),
    # function-level API (host values, device compute)
    "csattn_score_keys": (C.c_int, [vp, vp, u64, vp, vp, vp, u64, u64, C.c_int32, vp, vp]),
    "csattn_toplist_from_scores": (C.c_int, [vp, vp, u64, u64, vp, vp, vp]),
    "csattn_select_centroids": (C.c_int, [vp, vp, u64, vp, u64, vp, u64, C.c_double, vp, vp, vp, vp]),
    "csattn_reduce_by_key": (C.c_int, [vp, u64, vp, vp, vp, vp, vp, vp, vp, u64, vp]),
    "csattn_select_topk": (C.c_int, [vp, vp, vp, u64, u64, vp, u64, vp, vp]),
    "csattn_dense_attention_rows": (C.c_int, [vp, vp, vp, vp, u64, u64, vp, u64, vp, vp]),
    "csattn_dense_topk_rows": (C.c_int, [vp, vp, vp, u64, u64, u64, vp]),
    "csattn_ctx_set_kv_placement": (C.c_int, [vp, C.c_int32]),
    "csattn_f32_to_f16": (C.c_uint16, [C.c_float]),
    "csattn_f16_to_f32": (C.c_float, [C.c_uint16]),
    "csattn_csat_read_header": (C.c_int, [vp, u64, P(CsatHeaderC)]),
    "csattn_csat_footprint": (C.c_int, [P(CsatHeaderC), vp, P(u64), P(u64), P(u64)]),
    "csattn_csat_encode": (C.c_int, [P(CsatHeaderC), vp, vp, vp, vp, u64, vp, u64, P(u64)]),
    "csattn_csat_decode": (C.c_int, [vp, u64, P(CsatHeaderC), vp, vp, vp, vp, u64]),
    "csattn_session_serialize": (C.c_int, [vp, vp, u64, P(u64)]),
    "csattn_session_deserialize": (C.c_int, [vp, vp, u64, vp, vp, u64, P(RetrievalConfigC), u64, u64,
                                             P(vp)]),
    "csattn_session_gather_stats": (C.c_int, [vp, P(u64), P(u64)]),
    "csattn_session_fork": (C.c_int, [vp, u64, P(vp)]),
    "csattn_session_destroy": (C.c_int, [vp]),
    "csattn_session_info_get": (C.c_int, [vp, P(SessionInfoC)]),
    "csattn_session_set_retrieval": (C.c_int, [vp, P(RetrievalConfigC)]),
    "csattn_session_read_kv": (C.c_int, [vp, u64, u64, vp, vp]),
    "csattn_session_keep_candidates": (C.c_int, [vp, i32]),
    "csattn_session_candidates": (C.c_int, [vp, u64, vp, vp, u64, P(u64)]),
    "csattn_decode_step": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, u64, P(StepReportC), P(u64),
                                     u32]),
    "csattn_decode_batch": (C.c_int, [vp, u64, P(vp), vp, vp, vp, vp, vp, u64, u32]),
    "csattn_decode_run": (C.c_int, [vp, u64, P(vp), u64, vp, vp, vp, vp, vp, u64, vp, u32]),
    "csattn_dense_attention": (C.c_int, [vp, vp, vp, u64, vp, vp, u32]),
}


def header_symbols(path: str | None = None) -> list[str]:
    """Function names declared in include/csattn_b200.h."""
    import re
    path = path or os.path.join(os.path.dirname(_HERE), "include", "csattn_b200.h")
    text = open(path).read()
    return sorted(set(re.findall(r"\b(csattn_[a-z0-9_]+)\s*\(", text)))


_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the C ABI library, binding every declared symbol."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with __graft_entry__.build() "
            "(make -C paper_2604_08584_b200/csrc). There is no fallback path.")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
