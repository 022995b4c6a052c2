"""TEST INFRASTRUCTURE: ctypes mirrors of the plain-data structs of
include/csattn_b200.h that the checkers' C entry points take (oracle/ref_adapter.cpp
and oracle/csattn_oracle.c use the same header). Kept here so the oracle never
imports the product package: a bench reference arm maps only oracle/ libraries."""
import ctypes as C

STATUS_NAMES = {
    0: "ok", 1: "Error", 2: "DimensionError", 3: "ParameterError", 4: "DataError",
    5: "BadMagicError", 6: "VersionError", 7: "TruncatedError", 8: "CorruptError",
    9: "PropertyError", 10: "StreamExhaustedError", 20: "CudaError", 21: "CapacityError",
}


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


def as_struct(cls, x):
    """A checker-side copy of a same-layout struct built elsewhere (e.g. the
    product mirror's IndexConfig.c()); pointers inside are copied as values."""
    if isinstance(x, cls):
        return x
    if C.sizeof(x) != C.sizeof(cls):
        raise TypeError(f"{type(x).__name__} does not match {cls.__name__}")
    return cls.from_buffer_copy(x)
