"""TEST INFRASTRUCTURE ONLY: ctypes bindings of the two CPU checkers.

  * RefSession  — oracle/_ref/libcsattn_ref.so: the UNMODIFIED reference
                  library (built from /root/reference/proj/src by oracle/Makefile).
  * OraSession  — oracle/liboracle.so: the plain-C restatement (csattn_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
Both expose the same small session API as the product's Python mirror so a
parity test can drive all three on identical inputs.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from oracle import _cstructs as _abi

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libcsattn_ref.so")
ORA_LIB = os.path.join(HERE, "liboracle.so")

vp, u64, u32 = C.c_void_p, C.c_uint64, C.c_uint32
P = C.POINTER

_ref = None
_ora = None


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            raise RuntimeError(f"{REF_LIB} missing: run make -C oracle (needs /root/reference)")
        L = C.CDLL(REF_LIB)
        L.csref_last_error.restype = C.c_char_p
        L.csref_make_synthetic.argtypes = [P(_abi.SyntheticSpecC), vp, vp, vp]
        L.csref_mix_seed.restype = u64
        L.csref_mix_seed.argtypes = [u64, u64]
        L.csref_ceil_ratio.restype = u64
        L.csref_ceil_ratio.argtypes = [C.c_double, u64]
        L.csref_prefill.argtypes = [vp, u64, vp, vp, u64, u64, P(u64), u64,
                                    P(_abi.IndexConfigC), P(_abi.RetrievalConfigC), u64, P(vp)]
        L.csref_prefill_from_centroids.argtypes = [vp, u64, vp, vp, u64, u64, P(u64), u64,
                                                   P(_abi.IndexConfigC),
                                                   P(_abi.RetrievalConfigC), u64, P(vp)]
        L.csref_import.argtypes = [vp, u64, vp, vp, vp, u64, u64, C.c_double, C.c_int32, vp,
                                   vp, u64, u64, P(u64), u64, P(_abi.RetrievalConfigC), u64,
                                   P(vp)]
        L.csref_candidates.argtypes = [vp, u64, vp, vp, u64, P(u64)]
        L.csref_free.argtypes = [vp]
        L.csref_fork.argtypes = [vp, P(vp)]
        L.csref_set_retrieval.argtypes = [vp, P(_abi.RetrievalConfigC)]
        L.csref_info.argtypes = [vp, P(u64), P(u64), P(u64), P(u64)]
        L.csref_export.argtypes = [vp, vp, vp, vp, u64, vp]
        L.csref_step.argtypes = [vp, vp, vp, vp, vp, u64, vp, vp, P(_abi.StepReportC), P(u64)]
        L.csref_step_compare.argtypes = [vp, vp, vp, vp, vp, vp, vp, P(C.c_double),
                                         P(C.c_double)]
        L.csref_bench.argtypes = [P(vp), u64, vp, vp, vp, u64, u64, P(C.c_double)]
        L.csref_dense_attention.argtypes = [vp, vp, vp, u64, u64, vp, u64, vp, vp]
        L.csref_dense_topk.argtypes = [vp, vp, u64, u64, u64, vp]
        L.csref_f32_to_f16.restype = C.c_uint16
        L.csref_f32_to_f16.argtypes = [C.c_float]
        L.csref_f16_to_f32.restype = C.c_float
        L.csref_f16_to_f32.argtypes = [C.c_uint16]
        L.csref_encode.argtypes = [vp, u64, vp, vp, vp, u64, u64, u64, C.c_int32, C.c_int32, vp, u64,
                                   vp, u64, P(u64)]
        L.csref_serialize.argtypes = [vp, C.c_int32, vp, u64, P(u64)]
        L.csref_roundtrip.argtypes = [vp, u64, vp, u64, P(u64)]
        L.csref_footprint.argtypes = [vp, u64, P(u64), P(u64), P(u64)]
        L.csref_load.argtypes = [vp, u64, vp, vp, u64, vp, u64, P(vp)]
        _ref = L
    return _ref


def ora_lib():
    global _ora
    if _ora is None:
        if not os.path.exists(ORA_LIB):
            raise RuntimeError(f"{ORA_LIB} missing: run make -C oracle")
        L = C.CDLL(ORA_LIB)
        L.ora_mix_seed.restype = u64
        L.ora_mix_seed.argtypes = [u64, u64]
        L.ora_ceil_ratio.restype = u64
        L.ora_ceil_ratio.argtypes = [C.c_double, u64]
        L.ora_keep_count.argtypes = [C.c_double, u64, P(u64)]
        L.ora_dot.restype = C.c_double
        L.ora_dot.argtypes = [vp, vp, C.c_size_t]
        L.ora_l2_normalize.argtypes = [vp, C.c_size_t]
        L.ora_prefill.argtypes = [vp, u64, vp, vp, u64, u64, P(u64), u64, P(_abi.IndexConfigC),
                                  P(_abi.RetrievalConfigC), u64, P(vp)]
        L.ora_prefill_from_centroids.argtypes = [vp, u64, vp, vp, u64, u64, P(u64), u64,
                                                 P(_abi.IndexConfigC),
                                                 P(_abi.RetrievalConfigC), u64, P(vp)]
        L.ora_free.argtypes = [vp]
        L.ora_step.argtypes = [vp, vp, vp, vp, vp, u64, vp, vp, P(_abi.StepReportC)]
        L.ora_export.argtypes = [vp, vp, vp, vp, u64, vp]
        L.ora_context.restype = u64
        L.ora_context.argtypes = [vp]
        L.ora_attention.argtypes = [vp, vp, vp, C.c_size_t, C.c_size_t, vp, C.c_size_t, vp, vp]
        L.ora_select_topk.restype = C.c_size_t
        L.ora_select_topk.argtypes = [vp, vp, C.c_size_t, C.c_size_t, C.c_double, C.c_size_t,
                                      C.c_int, C.c_size_t, vp]
        L.ora_cosine_kmeans.argtypes = [vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                        C.c_size_t, u64, C.c_double, vp]
        L.ora_score_keys.argtypes = [vp, vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                     C.c_int, vp]
        _ora = L
    return _ora


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _rcfg(rcfg):
    """(checker-side RetrievalConfigC, weights array kept alive with it)"""
    rc, w = rcfg.c()
    return _abi.as_struct(_abi.RetrievalConfigC, rc), w


def _w(widths):
    return (C.c_uint64 * len(widths))(*[int(x) for x in widths])


class _Base:
    kind = ""

    def __init__(self, lib, h, d, group, n, L, T):
        self.lib, self.h, self.d, self.group, self.n, self.L, self.T = lib, h, d, group, n, L, T

    def step(self, q, key, value, want_weights=False):
        """One decode step for the group; returns list of (selected, out, weights, report)."""
        g, d, n = self.group, self.d, self.n
        q = _f32(q).reshape(g, d)
        key, value = _f32(key).reshape(d), _f32(value).reshape(d)
        sel = np.zeros((g, n), np.uint32)
        out = np.zeros((g, d), np.float32)
        wts = np.zeros((g, n), np.float32)
        reps = (_abi.StepReportC * g)()
        self._step(q, key, value, sel, n, out, wts, reps)
        self.n += 1
        res = []
        for h in range(g):
            k = int(reps[h].k)
            res.append((sel[h, :k].copy(), out[h].copy(), wts[h, :k].copy(), reps[h]))
        return res

    def export(self):
        T, L = self.T, max(self.L, 1)
        lens = np.zeros(T, np.uint32)
        idx = np.zeros((T, L), np.uint32)
        sc = np.zeros((T, L), np.float32)
        cent = np.zeros(self.C * self.d, np.float32)
        self._export(lens, idx, sc, L, cent)
        return lens, idx, sc, cent


class RefSession(_Base):
    """The reference library itself (GQA composition per oracle/ref_adapter.cpp)."""
    kind = "reference"

    @staticmethod
    def _chk(st):
        if st != 0:
            raise RuntimeError(f"reference error {_abi.STATUS_NAMES.get(st, st)}: "
                               f"{ref_lib().csref_last_error().decode()}")

    @classmethod
    def prefill(cls, queries, keys, values, widths, icfg, rcfg, group=1):
        L = ref_lib()
        d = sum(widths)
        q, k, v = _f32(queries), _f32(keys), _f32(values)
        ic = _abi.as_struct(_abi.IndexConfigC, icfg.c())
        rc, w = _rcfg(rcfg)
        h = C.c_void_p()
        st = L.csref_prefill(q.ctypes.data, q.size // d, k.ctypes.data, v.ctypes.data,
                             k.size // d, d, _w(widths), len(widths), C.byref(ic), C.byref(rc),
                             group, C.byref(h))
        cls._chk(st)
        return cls._wrap(h, d, group)

    @classmethod
    def from_centroids(cls, cent, keys, values, widths, icfg, rcfg, group=1):
        L = ref_lib()
        d = sum(widths)
        c = _f32(cent).reshape(-1)
        k, v = _f32(keys), _f32(values)
        ic = _abi.as_struct(_abi.IndexConfigC, icfg.c())
        rc, w = _rcfg(rcfg)
        h = C.c_void_p()
        st = L.csref_prefill_from_centroids(c.ctypes.data, c.size // d, k.ctypes.data,
                                            v.ctypes.data, k.size // d, d, _w(widths),
                                            len(widths), C.byref(ic), C.byref(rc), group,
                                            C.byref(h))
        cls._chk(st)
        return cls._wrap(h, d, group)

    @classmethod
    def load(cls, data, keys, values, d, rcfg, group=1):
        """load_index (deserialize_index) + KvStore + Session over the image."""
        a = np.frombuffer(bytes(data), np.uint8)
        k, v = _f32(keys), _f32(values)
        rc, w = _rcfg(rcfg)
        h = C.c_void_p()
        cls._chk(ref_lib().csref_load(a.ctypes.data, a.size, k.ctypes.data, v.ctypes.data, d,
                                      C.byref(rc), group, C.byref(h)))
        return cls._wrap(h, d, group)

    def serialize(self, score_bits=32):
        """serialize_index of the current index at the given score width."""
        n = C.c_uint64()
        self._chk(ref_lib().csref_serialize(self.h, score_bits, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        self._chk(ref_lib().csref_serialize(self.h, score_bits, buf, n.value, C.byref(n)))
        return bytes(buf)

    @classmethod
    def from_index(cls, cent, lens, idx, sc, L, alpha, keys, values, widths, rcfg, group=1,
                   normalize_keys=False):
        """A reference Session over a given CsIndex image (TopList order)."""
        d = sum(widths)
        c = _f32(cent).reshape(-1)
        lens = np.ascontiguousarray(lens, np.uint32)
        idx = np.ascontiguousarray(idx, np.uint32)
        sc = _f32(sc)
        k, v = _f32(keys), _f32(values)
        rc, w = _rcfg(rcfg)
        h = C.c_void_p()
        cls._chk(ref_lib().csref_import(c.ctypes.data, c.size // d, lens.ctypes.data,
                                        idx.ctypes.data, sc.ctypes.data, idx.shape[1], L, alpha,
                                        int(normalize_keys), k.ctypes.data, v.ctypes.data,
                                        k.size // d, d, _w(widths), len(widths), C.byref(rc),
                                        group, C.byref(h)))
        return cls._wrap(h, d, group)

    @classmethod
    def _wrap(cls, h, d, group):
        n, L, c, m = u64(), u64(), u64(), u64()
        ref_lib().csref_info(h, C.byref(n), C.byref(L), C.byref(c), C.byref(m))
        s = cls(ref_lib(), h, d, group, n.value, L.value, c.value * m.value)
        s.C = c.value
        s.m = m.value
        return s

    def set_retrieval(self, rcfg):
        rc, w = _rcfg(rcfg)
        self._keep_w = w
        self._chk(ref_lib().csref_set_retrieval(self.h, C.byref(rc)))

    def fork(self):
        """An independent copy (Session is a value type in the reference)."""
        h = C.c_void_p()
        self._chk(ref_lib().csref_fork(self.h, C.byref(h)))
        s = type(self)(self.lib, h, self.d, self.group, self.n, self.L, self.T)
        s.C, s.m = self.C, self.m
        return s

    def candidates(self, head=0):
        cap = self.n + 1
        idx = np.zeros(cap, np.uint32)
        sc = np.zeros(cap, np.float64)
        n = u64()
        self._chk(self.lib.csref_candidates(self.h, head, idx.ctypes.data, sc.ctypes.data, cap,
                                            C.byref(n)))
        return idx[:n.value].copy(), sc[:n.value].copy()

    def _step(self, q, key, value, sel, stride, out, wts, reps):
        self._chk(self.lib.csref_step(self.h, q.ctypes.data, key.ctypes.data, value.ctypes.data,
                                      sel.ctypes.data, stride, out.ctypes.data, wts.ctypes.data,
                                      reps, None))

    def _export(self, lens, idx, sc, stride, cent):
        self._chk(self.lib.csref_export(self.h, lens.ctypes.data, idx.ctypes.data,
                                        sc.ctypes.data, stride, cent.ctypes.data))

    def __del__(self):
        try:
            if self.h:
                self.lib.csref_free(self.h)
                self.h = None
        except Exception:
            pass


class OraSession(_Base):
    """The plain-C restatement."""
    kind = "port"

    @staticmethod
    def _chk(st):
        if st != 0:
            raise RuntimeError(f"oracle error {_abi.STATUS_NAMES.get(st, st)}")

    @classmethod
    def prefill(cls, queries, keys, values, widths, icfg, rcfg, group=1):
        L = ora_lib()
        d = sum(widths)
        q, k, v = _f32(queries), _f32(keys), _f32(values)
        ic = _abi.as_struct(_abi.IndexConfigC, icfg.c())
        rc, w = _rcfg(rcfg)
        h = C.c_void_p()
        cls._chk(L.ora_prefill(q.ctypes.data, q.size // d, k.ctypes.data, v.ctypes.data,
                               k.size // d, d, _w(widths), len(widths), C.byref(ic),
                               C.byref(rc), group, C.byref(h)))
        s = cls._wrap(h, d, group, icfg.centroids, len(widths), k.size // d, icfg)
        s._keep = w
        return s

    @classmethod
    def from_centroids(cls, cent, keys, values, widths, icfg, rcfg, group=1):
        L = ora_lib()
        d = sum(widths)
        c = _f32(cent).reshape(-1)
        k, v = _f32(keys), _f32(values)
        ic = _abi.as_struct(_abi.IndexConfigC, icfg.c())
        rc, w = _rcfg(rcfg)
        h = C.c_void_p()
        cls._chk(L.ora_prefill_from_centroids(c.ctypes.data, c.size // d, k.ctypes.data,
                                              v.ctypes.data, k.size // d, d, _w(widths),
                                              len(widths), C.byref(ic), C.byref(rc), group,
                                              C.byref(h)))
        s = cls._wrap(h, d, group, c.size // d, len(widths), k.size // d, icfg)
        s._keep = w
        return s

    @classmethod
    def _wrap(cls, h, d, group, c, m, p, icfg):
        Lc = icfg.list_capacity or ora_lib().ora_ceil_ratio(icfg.alpha, p)
        s = cls(ora_lib(), h, d, group, p, Lc, c * m)
        s.C = c
        s.m = m
        return s

    def _step(self, q, key, value, sel, stride, out, wts, reps):
        self._chk(self.lib.ora_step(self.h, q.ctypes.data, key.ctypes.data, value.ctypes.data,
                                    sel.ctypes.data, stride, out.ctypes.data, wts.ctypes.data,
                                    reps))

    def _export(self, lens, idx, sc, stride, cent):
        self._chk(self.lib.ora_export(self.h, lens.ctypes.data, idx.ctypes.data,
                                      sc.ctypes.data, stride, cent.ctypes.data))

    def __del__(self):
        try:
            if self.h:
                self.lib.ora_free(self.h)
                self.h = None
        except Exception:
            pass


def ref_bench(sessions, q, k, v, steps, threads):
    """Wall seconds for `steps` decode steps of every session on `threads` host
    threads. q: [n, steps, group, d]; k, v: [n, steps, d] (float32)."""
    n = len(sessions)
    hs = (C.c_void_p * n)(*[s.h.value if isinstance(s.h, C.c_void_p) else s.h for s in sessions])
    q, k, v = _f32(q), _f32(k), _f32(v)
    sec = C.c_double()
    RefSession._chk(ref_lib().csref_bench(hs, n, q.ctypes.data, k.ctypes.data, v.ctypes.data,
                                          steps, threads, C.byref(sec)))
    for s in sessions:
        s.n += steps
    return sec.value


def ref_make_synthetic(spec):
    q = np.empty((spec.rows, spec.dim), np.float32)
    k = np.empty_like(q)
    v = np.empty_like(q)
    s = _abi.SyntheticSpecC(spec.rows, spec.dim, spec.clusters, spec.seed, spec.plant_fraction,
                            spec.plant_scale, spec.query_noise, spec.dwell)
    st = ref_lib().csref_make_synthetic(C.byref(s), q.ctypes.data, k.ctypes.data, v.ctypes.data)
    if st:
        raise RuntimeError("make_synthetic failed")
    return q, k, v
