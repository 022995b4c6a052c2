"""B200-native CSAttention decode hot path (arXiv 2604.08584), Python host mirror.

The product is libcsattn_b200.so: sm_100a kernels behind the C ABI in
include/csattn_b200.h. This module mirrors the reference C++ API of
proj/include/csattn/ (same names, argument meaning and error classes) on top
of that ABI, so parity tests read like the reference's own tests:

    reference (C++)                      here
    ---------------------------------    -------------------------------------
    prefill  (session.hpp:46-49)         prefill(ctx, q, k, v, widths, icfg, cfg)
    build_index_from_centroids (:92-96)  prefill_from_centroids(...)
    decode_step (session.hpp:54-57)      Session.decode_step(q, k, v)
    run_decode  (session.hpp:61-66)      run_decode(session, qs, ks, vs, steps)
    keep_count / parse_schedule          keep_count / parse_schedule
    make_synthetic (synthetic.hpp:38-41) make_synthetic(SyntheticSpec)
    Error / DimensionError / ...         same exception classes

Host buffers are numpy arrays (copied in/out inside the call); torch CUDA
tensors are passed as device pointers.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi

__all__ = [
    "Error", "DimensionError", "ParameterError", "DataError", "BadMagicError", "VersionError",
    "TruncatedError", "CorruptError", "PropertyError", "StreamExhaustedError", "CudaError",
    "CapacityError", "IndexConfig", "RetrievalConfig", "SyntheticSpec", "CostCounters",
    "DecodeStepReport", "Context", "Session", "prefill", "prefill_batch", "prefill_from_centroids",
    "import_index", "run_decode", "keep_count", "parse_schedule", "h2d_bytes", "make_synthetic",
    "uniform_widths", "lib",
]


# ---- exceptions (errors.hpp:8-52) ----
class Error(RuntimeError):
    pass


class DimensionError(Error):
    pass


class ParameterError(Error):
    pass


class DataError(Error):
    pass


class BadMagicError(DataError):
    pass


class VersionError(DataError):
    pass


class TruncatedError(DataError):
    pass


class CorruptError(DataError):
    pass


class PropertyError(Error):
    pass


class StreamExhaustedError(Error):
    pass


class CudaError(Error):
    pass


class CapacityError(ParameterError):
    pass


_EXC = {1: Error, 2: DimensionError, 3: ParameterError, 4: DataError, 5: BadMagicError,
        6: VersionError, 7: TruncatedError, 8: CorruptError, 9: PropertyError,
        10: StreamExhaustedError, 20: CudaError, 21: CapacityError}


def lib():
    return _abi.load()


def _check(status: int) -> None:
    if status != 0:
        msg = lib().csattn_last_error().decode()
        raise _EXC.get(status, Error)(msg)


# ---- configs (index.hpp:36-42, clustering.hpp:17-28, retrieval.hpp:17-32) ----
@dataclass
class IndexConfig:
    alpha: float = 0.2
    list_capacity: int = 0
    normalize_keys: bool = False
    score_bits: int = 16
    centroids: int = 64
    iterations: int = 10
    batch_size: int = 0
    seed: int = 0
    tolerance: float = 1e-7

    def c(self) -> _abi.IndexConfigC:
        return _abi.IndexConfigC(self.alpha, self.list_capacity, int(self.normalize_keys),
                                 self.score_bits, self.centroids, self.iterations,
                                 self.batch_size, self.seed, self.tolerance)


@dataclass
class RetrievalConfig:
    keep_ratio: float = 0.05
    search_period: int = 1
    recent_window: int = 32
    weights: list = field(default_factory=list)
    backoff_tau: int = 1
    backoff_threshold: float = -math.inf
    recent_passthrough: bool = True

    def c(self):
        w = np.ascontiguousarray(self.weights, dtype=np.float64)
        cfg = _abi.RetrievalConfigC(
            self.keep_ratio, self.search_period, self.recent_window,
            w.ctypes.data_as(C.POINTER(C.c_double)) if len(w) else None, len(w),
            self.backoff_tau, self.backoff_threshold, int(self.recent_passthrough), 0)
        return cfg, w  # keep w alive with the struct


@dataclass
class SyntheticSpec:
    rows: int = 0
    dim: int = 64
    clusters: int = 8
    seed: int = 0
    plant_fraction: float = 0.08
    plant_scale: float = 6.0
    query_noise: float = 0.05
    dwell: int = 32


@dataclass
class CostCounters:
    centroid_dot_ops: int = 0
    gathered_entries: int = 0
    reduce_ops: int = 0
    attention_key_ops: int = 0
    h2d_bytes_model: float = 0.0
    searches: int = 0
    inserts_attempted: int = 0
    inserts_applied: int = 0
    insert_dot_ops: int = 0


@dataclass
class DecodeStepReport:
    selected: np.ndarray
    k: int
    searched: bool
    output: np.ndarray
    weights: np.ndarray | None
    counters: CostCounters
    worst_best_cosine: float = 1.0


# ---- small pure helpers ----
def keep_count(rho: float, n: int) -> int:
    out = C.c_uint64()
    _check(lib().csattn_keep_count(rho, n, C.byref(out)))
    return out.value


def parse_schedule(name: str) -> tuple[float, int]:
    rho, per = C.c_double(), C.c_uint64()
    _check(lib().csattn_parse_schedule(name.encode(), C.byref(rho), C.byref(per)))
    return rho.value, per.value


def h2d_bytes(rho: float, n: int, d: int, b: int, period: int) -> float:
    out = C.c_double()
    _check(lib().csattn_h2d_bytes(rho, n, d, b, period, C.byref(out)))
    return out.value


def uniform_widths(dim: int, subspaces: int) -> list[int]:
    """SubspaceLayout::uniform (core.cpp:35-41)."""
    if subspaces == 0 or subspaces > dim:
        raise ParameterError("uniform layout requires 1 <= m <= d")
    w = [dim // subspaces] * subspaces
    for b in range(dim % subspaces):
        w[b] += 1
    return w


def make_synthetic(spec: SyntheticSpec):
    """make_synthetic (synthetic.cpp:18-74): returns (queries, keys, values) rows x dim f32."""
    q = np.empty((spec.rows, spec.dim), np.float32)
    k = np.empty_like(q)
    v = np.empty_like(q)
    s = _abi.SyntheticSpecC(spec.rows, spec.dim, spec.clusters, spec.seed, spec.plant_fraction,
                            spec.plant_scale, spec.query_noise, spec.dwell)
    _check(lib().csattn_make_synthetic(C.byref(s), q.ctypes.data, k.ctypes.data, v.ctypes.data))
    return q, k, v


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _is_cuda(t) -> bool:
    return hasattr(t, "is_cuda") and t.is_cuda


def _ptr(t):
    """(pointer, is_host) for a numpy array or torch tensor."""
    if t is None:
        return None, True
    if _is_cuda(t):
        return C.c_void_p(t.data_ptr()), False
    if hasattr(t, "numpy"):
        t = t.numpy()
    return C.c_void_p(t.ctypes.data), True


class Context:
    """A CUDA device + stream (csattn_ctx)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        h = C.c_void_p()
        _check(lib().csattn_ctx_create(device, C.c_void_p(stream) if stream else None,
                                       C.byref(h)))
        self.h = h
        self.device = device

    def set_kv_placement(self, placement: str):
        """'device' (HBM, default) or 'host': sessions created afterwards keep
        their KV rows in mapped pinned host memory (offload mode)."""
        _check(lib().csattn_ctx_set_kv_placement(self.h, {"device": 0, "host": 1}[placement]))

    def synchronize(self):
        _check(lib().csattn_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        return lib().csattn_ctx_launch_count(self.h)

    @property
    def build_stats(self) -> tuple:
        """(table builds through the tcgen05 screen, of those rebuilt by the
        plain fp64 kernels because a table's screen was inconclusive)."""
        a, b = C.c_uint64(), C.c_uint64()
        _check(lib().csattn_ctx_build_stats(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def profile(self, enable: bool = True):
        """Bracket every decode / insert launch with CUDA events on this stream."""
        _check(lib().csattn_ctx_profile(self.h, int(enable)))

    def profile_read(self, reset: bool = True) -> dict:
        ms = (C.c_double * 3)()
        n = C.c_uint64()
        _check(lib().csattn_ctx_profile_read(self.h, ms, C.byref(n), int(reset)))
        return {"select_ms": ms[0], "attend_ms": ms[1], "insert_ms": ms[2], "steps": n.value}

    def close(self):
        if self.h:
            lib().csattn_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Session:
    """One KV head's prefill -> decode lifecycle (session.hpp:19-31), device resident."""

    def __init__(self, ctx: Context, handle: C.c_void_p):
        self.ctx = ctx
        self.h = handle

    # -- introspection --
    def info(self) -> _abi.SessionInfoC:
        i = _abi.SessionInfoC()
        _check(lib().csattn_session_info_get(self.h, C.byref(i)))
        return i

    @property
    def context_len(self) -> int:
        return self.info().context_len

    @property
    def group(self) -> int:
        return self.info().group

    def export_index(self):
        """(lens[T], indices[T,L], scores[T,L], centroids[C*d]) in TopList order."""
        inf = self.info()
        T = inf.subspaces * inf.centroids
        L = inf.list_capacity
        lens = np.zeros(T, np.uint32)
        idx = np.zeros((T, max(L, 1)), np.uint32)
        sc = np.zeros((T, max(L, 1)), np.float32)
        cent = np.zeros(inf.centroids * inf.dim, np.float32)
        _check(lib().csattn_session_export(self.h, lens.ctypes.data, idx.ctypes.data,
                                           sc.ctypes.data, max(L, 1), cent.ctypes.data))
        return lens, idx, sc, cent

    def read_kv(self, first: int = 0, count: int | None = None):
        inf = self.info()
        if count is None:
            count = inf.context_len - first
        k = np.zeros((count, inf.dim), np.float32)
        v = np.zeros_like(k)
        _check(lib().csattn_session_read_kv(self.h, first, count, k.ctypes.data, v.ctypes.data))
        return k, v

    def keep_candidates(self, enable: bool = True):
        """Keep every search's CandidateSet on the device (SearchState::cached)."""
        _check(lib().csattn_session_keep_candidates(self.h, int(enable)))

    def candidates(self, head: int = 0):
        """(indices ascending, fp64 scores) of the last search of `head`."""
        cap = self.info().max_context
        idx = np.zeros(cap, np.uint32)
        sc = np.zeros(cap, np.float64)
        n = C.c_uint64()
        _check(lib().csattn_session_candidates(self.h, head, idx.ctypes.data, sc.ctypes.data,
                                               cap, C.byref(n)))
        return idx[:n.value].copy(), sc[:n.value].copy()

    def fork(self, max_decode_steps: int | None = None) -> "Session":
        inf = self.info()
        if max_decode_steps is None:
            max_decode_steps = inf.max_context - inf.prefill_len
        h = C.c_void_p()
        _check(lib().csattn_session_fork(self.h, max_decode_steps, C.byref(h)))
        return Session(self.ctx, h)

    def set_retrieval(self, cfg: RetrievalConfig):
        c, w = cfg.c()
        _check(lib().csattn_session_set_retrieval(self.h, C.byref(c)))

    # -- decode (session.cpp:46-99) --
    def decode_step(self, q, new_key, new_value, want_weights: bool = False,
                    k_override=None) -> DecodeStepReport | list[DecodeStepReport]:
        inf = self.info()
        g, d, n = inf.group, inf.dim, inf.context_len
        q = _f32(q).reshape(g, d)
        nk = _f32(new_key).reshape(d)
        nv = _f32(new_value).reshape(d)
        if q.shape[1] != d or nk.shape[0] != d or nv.shape[0] != d:
            raise DimensionError("decode step inputs must have width d")
        out = np.zeros((g, d), np.float32)
        sel = np.zeros((g, n), np.uint32)
        wts = np.zeros((g, n), np.float32) if want_weights else None
        reps = (_abi.StepReportC * g)()
        ko = None
        if k_override is not None:
            ko = (C.c_uint64 * g)(*([int(x) for x in np.atleast_1d(k_override)]))
        _check(lib().csattn_decode_step(
            self.h, q.ctypes.data, nk.ctypes.data, nv.ctypes.data, out.ctypes.data,
            sel.ctypes.data, wts.ctypes.data if wts is not None else None, n, reps, ko,
            _abi.HOST_BUFFERS))
        res = []
        for h in range(g):
            r = reps[h]
            k = int(r.k)
            res.append(DecodeStepReport(
                selected=sel[h, :k].copy(), k=k, searched=bool(r.searched), output=out[h].copy(),
                weights=wts[h, :k].copy() if wts is not None else None,
                counters=CostCounters(r.centroid_dot_ops, r.gathered_entries, r.reduce_ops,
                                      r.attention_key_ops, r.h2d_bytes_model, r.searches,
                                      r.inserts_attempted, r.inserts_applied, r.insert_dot_ops),
                worst_best_cosine=r.worst_best_cosine))
        return res[0] if g == 1 else res

    # -- the dense oracle on the device (core.cpp:118-192) --
    def dense_attention(self, q, mask=None):
        """Masked (mask = row indices) or full dense_attention over the current
        KV rows: (output[d], weights[len(mask) or N])."""
        inf = self.info()
        qv = _f32(q).reshape(inf.dim)
        n = inf.context_len if mask is None else len(mask)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint32)
        out = np.zeros(inf.dim, np.float32)
        w = np.zeros(max(n, 1), np.float32)
        _check(lib().csattn_dense_attention(self.h, qv.ctypes.data, None if m is None else m.ctypes.data,
                                            0 if m is None else m.size, out.ctypes.data, w.ctypes.data,
                                            _abi.HOST_BUFFERS))
        return out, w[:n]

    def dense_topk(self, q, k: int) -> np.ndarray:
        """dense_topk: the k best rows by sequential-fp64 q.k, ascending."""
        qv = _f32(q).reshape(self.info().dim)
        out = np.zeros(max(int(k), 1), np.uint32)
        _check(lib().csattn_dense_topk(self.h, qv.ctypes.data, int(k), out.ctypes.data, _abi.HOST_BUFFERS))
        return out[:int(k)]

    # -- CSAT v1 image (serialize_index, index.cpp:289-318) --
    def serialize(self) -> bytes:
        """The session's current index as a CSAT v1 image (tables ordered and
        encoded on the device)."""
        n = C.c_uint64()
        _check(lib().csattn_session_serialize(self.h, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        _check(lib().csattn_session_serialize(self.h, buf, n.value, C.byref(n)))
        return bytes(buf)

    def close(self):
        if self.h:
            lib().csattn_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def decode_batch(sessions, q, new_keys, new_values):
    """One decode step for a batch of sessions on one context (csattn_decode_batch):
    q holds sum(group) query rows in session order, new_keys/new_values one row
    per session. Returns (out [rows, d], selected [rows, max context]); row r's
    selected set is selected[r, :k] with k = keep_count(keep_ratio, context)."""
    if not sessions:
        raise ParameterError("no sessions")
    ctx = sessions[0].ctx
    d = sessions[0].info().dim
    rows = sum(s.group for s in sessions)
    stride = max(s.context_len for s in sessions)
    q = _f32(q).reshape(rows, d)
    nk = _f32(new_keys).reshape(len(sessions), d)
    nv = _f32(new_values).reshape(len(sessions), d)
    out = np.zeros((rows, d), np.float32)
    sel = np.zeros((rows, stride), np.uint32)
    hs = (C.c_void_p * len(sessions))(*[s.h for s in sessions])
    _check(lib().csattn_decode_batch(ctx.h, len(sessions), hs, q.ctypes.data, nk.ctypes.data,
                                     nv.ctypes.data, out.ctypes.data, sel.ctypes.data, stride,
                                     _abi.HOST_BUFFERS))
    return out, sel


def decode_run(sessions, q, new_keys, new_values, k_override=None):
    """run_decode over T steps of a session set as ONE CUDA graph
    (csattn_decode_run; session.cpp:101-126 without the per-step reports):
    q is [T, rows, d], new_keys/new_values [T, len(sessions), d] — numpy arrays
    (host) or CUDA tensors (device, outputs returned as CUDA tensors).
    k_override, if given, is [T, rows] (0 = keep_count). Returns (out [T, rows,
    d], selected [T, rows, stride]); step t's row r set is selected[t, r, :k]
    with k its keep count. Equal to T calls of decode_batch."""
    if not sessions:
        raise ParameterError("no sessions")
    ctx = sessions[0].ctx
    d = sessions[0].info().dim
    rows = sum(s.group for s in sessions)
    ns = len(sessions)
    T = int(q.shape[0])
    stride = max(s.context_len for s in sessions) + T
    ko = None
    if k_override is not None:
        ko = np.ascontiguousarray(np.asarray(k_override, dtype=np.uint64).reshape(T, rows))
    hs = (C.c_void_p * ns)(*[s.h for s in sessions])
    if _is_cuda(q):
        import torch
        q = q.contiguous().float()
        nk = new_keys.contiguous().float()
        nv = new_values.contiguous().float()
        if tuple(q.shape) != (T, rows, d) or nk.numel() != T * ns * d or nv.numel() != T * ns * d:
            raise DimensionError("decode_run: q [T, rows, d], keys/values [T, sessions, d]")
        out = torch.empty((T, rows, d), dtype=torch.float32, device=q.device)
        sel = torch.empty((T, rows, stride), dtype=torch.int32, device=q.device)
        torch.cuda.current_stream(q.device).synchronize()  # inputs ready for the context's stream
        _check(lib().csattn_decode_run(ctx.h, ns, hs, T, q.data_ptr(), nk.data_ptr(),
                                       nv.data_ptr(), out.data_ptr(), sel.data_ptr(), stride,
                                       ko.ctypes.data if ko is not None else None, 0))
        return out, sel
    q = _f32(q).reshape(T, rows, d)
    nk = _f32(new_keys).reshape(T, ns, d)
    nv = _f32(new_values).reshape(T, ns, d)
    out = np.zeros((T, rows, d), np.float32)
    sel = np.zeros((T, rows, stride), np.uint32)
    _check(lib().csattn_decode_run(ctx.h, ns, hs, T, q.ctypes.data, nk.ctypes.data,
                                   nv.ctypes.data, out.ctypes.data, sel.ctypes.data, stride,
                                   ko.ctypes.data if ko is not None else None,
                                   _abi.HOST_BUFFERS))
    return out, sel


def _widths_arr(widths):
    return (C.c_uint64 * len(widths))(*[int(w) for w in widths])


def prefill(ctx: Context, queries, keys, values, widths, index_cfg: IndexConfig,
            cfg: RetrievalConfig, group: int = 1, max_decode_steps: int = 1024) -> Session:
    """prefill (session.cpp:25-44) with the GPU table build; queries may pool a GQA group."""
    d = sum(widths)
    qp, qh = _ptr(queries)
    kp, kh = _ptr(keys)
    vp_, vh = _ptr(values)
    if not (qh == kh == vh):
        raise ParameterError("queries/keys/values must all be host arrays or all CUDA tensors")
    if qh:
        queries, keys, values = _f32(queries), _f32(keys), _f32(values)
        qp, kp, vp_ = (C.c_void_p(a.ctypes.data) for a in (queries, keys, values))
    nq = int(np.prod(queries.shape)) // d if d else 0
    p = int(np.prod(keys.shape)) // d if d else 0
    if d == 0 or int(np.prod(queries.shape)) % d or int(np.prod(keys.shape)) % d:
        raise DimensionError("prefill rows are not a multiple of d")
    if int(np.prod(values.shape)) != int(np.prod(keys.shape)):
        raise DimensionError("prefill key/value counts differ")
    ic = index_cfg.c()
    rc, w = cfg.c()
    h = C.c_void_p()
    _check(lib().csattn_prefill(ctx.h, qp, nq, kp, vp_, p, d, _widths_arr(widths), len(widths),
                                C.byref(ic), C.byref(rc), group, max_decode_steps,
                                _abi.HOST_BUFFERS if qh else 0, C.byref(h)))
    return Session(ctx, h)


def prefill_batch(ctx: Context, rows, widths, index_cfg, cfg: RetrievalConfig,
                  group: int = 1, max_decode_steps: int = 1024) -> list[Session]:
    """A layer's prefill (csattn_prefill_batch): rows = [(queries, keys, values), ...]
    as host arrays, one entry per KV head; index_cfg is one IndexConfig or one per
    entry. One k-means launch for all of them; session i equals
    prefill(ctx, *rows[i], widths, index_cfg[i], ...)."""
    cfgs = list(index_cfg) if isinstance(index_cfg, (list, tuple)) else [index_cfg] * len(rows)
    if len(cfgs) != len(rows):
        raise ParameterError("one index config per prefill entry")
    d = sum(widths)
    keep, arr = [], (_abi.PrefillRowsC * len(rows))()
    for i, (q, k, v) in enumerate(rows):
        q, k, v = _f32(q), _f32(k), _f32(v)
        if d == 0 or q.size % d or k.size % d:
            raise DimensionError("prefill rows are not a multiple of d")
        if v.size != k.size:
            raise DimensionError("prefill key/value counts differ")
        keep += [q, k, v]
        arr[i] = _abi.PrefillRowsC(q.ctypes.data, q.size // d, k.ctypes.data, v.ctypes.data,
                                   k.size // d)
    ics = (_abi.IndexConfigC * len(rows))(*[c.c() for c in cfgs])
    rc, w = cfg.c()
    hs = (C.c_void_p * len(rows))()
    _check(lib().csattn_prefill_batch(ctx.h, len(rows), arr, d, _widths_arr(widths), len(widths),
                                      ics, C.byref(rc), group, max_decode_steps,
                                      _abi.HOST_BUFFERS, hs))
    return [Session(ctx, C.c_void_p(h)) for h in hs]


def prefill_from_centroids(ctx: Context, centroids, keys, values, widths,
                           index_cfg: IndexConfig, cfg: RetrievalConfig, group: int = 1,
                           max_decode_steps: int = 1024) -> Session:
    """build_index_from_centroids (index.cpp:179-202): centroids packed per subspace (C*d)."""
    d = sum(widths)
    cent = _f32(centroids).reshape(-1)
    c = cent.size // d if d else 0
    keys, values = _f32(keys), _f32(values)
    if d == 0 or keys.size % d:
        raise DimensionError("prefill rows are not a multiple of d")
    if values.size != keys.size:
        raise DimensionError("prefill key/value counts differ")
    ic = index_cfg.c()
    rc, w = cfg.c()
    h = C.c_void_p()
    _check(lib().csattn_prefill_from_centroids(
        ctx.h, cent.ctypes.data, c, keys.ctypes.data, values.ctypes.data, keys.size // d, d,
        _widths_arr(widths), len(widths), C.byref(ic), C.byref(rc), group, max_decode_steps,
        _abi.HOST_BUFFERS, C.byref(h)))
    return Session(ctx, h)


def import_index(ctx: Context, centroids, lens, indices, scores, list_capacity: int,
                 alpha: float, keys, values, widths, cfg: RetrievalConfig, group: int = 1,
                 max_decode_steps: int = 1024, normalize_keys: bool = False,
                 score_bits: int = 32) -> Session:
    """Adopt a host CsIndex image (TopList order) as a device session."""
    d = sum(widths)
    cent = _f32(centroids).reshape(-1)
    lens = np.ascontiguousarray(lens, np.uint32)
    idx = np.ascontiguousarray(indices, np.uint32)
    sc = _f32(scores)
    keys, values = _f32(keys), _f32(values)
    rc, w = cfg.c()
    h = C.c_void_p()
    _check(lib().csattn_session_import(
        ctx.h, cent.ctypes.data, cent.size // d, lens.ctypes.data, idx.ctypes.data,
        sc.ctypes.data, idx.shape[1], list_capacity, alpha, int(normalize_keys), score_bits,
        keys.ctypes.data, values.ctypes.data, keys.size // d, d, _widths_arr(widths),
        len(widths), C.byref(rc), group, max_decode_steps, C.byref(h)))
    return Session(ctx, h)


def recall_at_k(selected, truth) -> float:
    """recall_at_k (metrics.cpp:9-30): |selected & truth| / |truth|."""
    truth = np.asarray(truth)
    if truth.size == 0:
        raise ParameterError("recall is undefined against an empty truth set")
    return float(np.intersect1d(np.asarray(selected), truth).size) / float(truth.size)


# ---- CSAT v1 index images (index.hpp:98-121) ----

def f32_to_f16(x: float) -> int:
    return int(lib().csattn_f32_to_f16(float(x)))


def f16_to_f32(h: int) -> float:
    return float(lib().csattn_f16_to_f32(int(h)))


def _u8(data):
    a = np.frombuffer(bytes(data), dtype=np.uint8)
    return a, (a.ctypes.data if a.size else None)


def csat_header(data) -> dict:
    """Header fields of a CSAT image (deserialize_index's checks through the widths)."""
    a, p = _u8(data)
    h = _abi.CsatHeaderC()
    _check(lib().csattn_csat_read_header(p, a.size, C.byref(h)))
    return dict(m=h.m, centroids=h.centroids, list_capacity=h.list_capacity, dim=h.dim,
                prefill_len=h.prefill_len, score_bits=h.score_bits,
                normalize_keys=bool(h.normalize_keys), widths=list(h.widths[:h.m]))


def _header_c(hd: dict):
    h = _abi.CsatHeaderC()
    h.m, h.centroids, h.list_capacity = hd["m"], hd["centroids"], hd["list_capacity"]
    h.dim, h.prefill_len, h.score_bits = hd["dim"], hd["prefill_len"], hd["score_bits"]
    h.normalize_keys = int(hd["normalize_keys"])
    for b, w in enumerate(hd["widths"]):
        h.widths[b] = w
    return h


def csat_decode(data):
    """deserialize_index on the host: (header dict, centroids, lens, indices, scores)."""
    a, p = _u8(data)
    hd = csat_header(data)
    T, L = hd["m"] * hd["centroids"], hd["list_capacity"]
    cent = np.zeros(hd["centroids"] * hd["dim"], np.float32)
    lens = np.zeros(T, np.uint32)
    ix = np.zeros((T, L), np.uint32)
    sc = np.zeros((T, L), np.float32)
    h = _abi.CsatHeaderC()
    _check(lib().csattn_csat_decode(p, a.size, C.byref(h), cent.ctypes.data, lens.ctypes.data,
                                    ix.ctypes.data, sc.ctypes.data, L))
    return hd, cent, lens, ix, sc


def csat_encode(header: dict, centroids, lens, indices, scores) -> bytes:
    """serialize_index of host tables in TopList order (rows of `indices`/`scores`)."""
    h = _header_c(header)
    cent = _f32(centroids).ravel()
    lens = np.ascontiguousarray(lens, np.uint32)
    ix = np.ascontiguousarray(indices, np.uint32)
    sc = np.ascontiguousarray(scores, np.float32)
    stride = ix.shape[1] if ix.ndim == 2 else ix.size
    n = C.c_uint64()
    _check(lib().csattn_csat_encode(C.byref(h), cent.ctypes.data, lens.ctypes.data, ix.ctypes.data,
                                    sc.ctypes.data, stride, None, 0, C.byref(n)))
    buf = (C.c_uint8 * n.value)()
    _check(lib().csattn_csat_encode(C.byref(h), cent.ctypes.data, lens.ctypes.data, ix.ctypes.data,
                                    sc.ctypes.data, stride, buf, n.value, C.byref(n)))
    return bytes(buf)


def csat_footprint(header: dict, lens) -> dict:
    """index_footprint (index.cpp:419-431)."""
    h = _header_c(header)
    lens = np.ascontiguousarray(lens, np.uint32)
    a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
    _check(lib().csattn_csat_footprint(C.byref(h), lens.ctypes.data, C.byref(a), C.byref(b), C.byref(c)))
    return dict(header_bytes=a.value, centroid_bytes=b.value, entry_bytes=c.value,
                payload=b.value + c.value, total=a.value + b.value + c.value)


def deserialize(ctx: Context, data, keys, values, cfg: RetrievalConfig, group: int = 1,
                max_decode_steps: int = 4096) -> Session:
    """A session from a CSAT image and the prefill KV rows it indexes
    (load_index + KvStore + Session, session.hpp:19-31)."""
    a, p = _u8(data)
    k = _f32(keys)
    v = _f32(values)
    hd = csat_header(data)
    rows = k.size // hd["dim"] if hd["dim"] else 0
    rc, w = cfg.c()
    h = C.c_void_p()
    _check(lib().csattn_session_deserialize(ctx.h, p, a.size, k.ctypes.data, v.ctypes.data, rows,
                                            C.byref(rc), group, max_decode_steps, C.byref(h)))
    return Session(ctx, h)


def run_decode(session: Session, queries, keys, values, steps: int,
               want_weights: bool = False) -> list:
    """run_decode (session.cpp:101-126): validates stream lengths up front."""
    inf = session.info()
    d, g = inf.dim, inf.group
    queries, keys, values = _f32(queries), _f32(keys), _f32(values)
    if queries.size % d or keys.size % d or values.size % d:
        raise DimensionError("decode rows are not a multiple of d")
    available = min(queries.size // (d * g), keys.size // d, values.size // d)
    if available < steps:
        raise StreamExhaustedError(f"decode streams run out at step {available} of {steps}")
    q = queries.reshape(-1, g * d)
    k = keys.reshape(-1, d)
    v = values.reshape(-1, d)
    return [session.decode_step(q[t], k[t], v[t], want_weights) for t in range(steps)]
