"""The dense oracle on the device: dense_topk
(core.cpp:171-192) exactly equal to the reference's, including appended rows
and exact score ties; masked and full dense_attention (core.cpp:118-169)
within fp64-rounding distance of the reference's; validation messages."""
import ctypes as C

import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from oracle import bindings as ob
from tests.helpers import rel_err, workload

pytestmark = pytest.mark.gpu


def _ref_topk(q, keys, k):
    n, d = keys.shape
    out = np.zeros(k, np.uint32)
    assert ob.ref_lib().csref_dense_topk(q.ctypes.data, keys.ctypes.data, n, d, k, out.ctypes.data) == 0
    return out


def _ref_attention(q, keys, values, mask=None):
    n, d = keys.shape
    m = None if mask is None else np.ascontiguousarray(mask, np.uint32)
    cnt = n if m is None else m.size
    out = np.zeros(d, np.float32)
    w = np.zeros(cnt, np.float32)
    st = ob.ref_lib().csref_dense_attention(q.ctypes.data, keys.ctypes.data, values.ctypes.data, n, d,
                                            None if m is None else m.ctypes.data, 0 if m is None else m.size,
                                            out.ctypes.data, w.ctypes.data)
    assert st == 0
    return out, w


def _session(ctx, P, T, d, seed, dup=False):
    q, k, v = workload(P, T, d, seed=seed)
    if dup:  # exact score ties: repeated key rows
        k[P // 2:P // 2 + 64] = k[10]
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=32)
    g = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, cs.RetrievalConfig(), max_decode_steps=T)
    for t in range(T):  # appended rows live in the session's tail store
        g.decode_step(q[P + t], k[P + t], v[P + t])
    return g, q, k[:P + T], v[:P + T]


@pytest.mark.parametrize("dup", [False, True])
def test_dense_topk_equals_reference(ctx, dup):
    g, q, k, v = _session(ctx, 20000, 8, 64, seed=41, dup=dup)
    rng = np.random.default_rng(3)
    for trial in range(6):
        qq = q[rng.integers(len(q))] if trial % 2 else k[10] * 0.5  # ties when dup
        for kk in (1, 37, 1001, len(k)):
            assert np.array_equal(g.dense_topk(qq, kk), _ref_topk(np.ascontiguousarray(qq), k, kk)), (trial, kk)


def test_dense_attention_matches_reference(ctx):
    g, q, k, v = _session(ctx, 12000, 6, 64, seed=42)
    rng = np.random.default_rng(4)
    for trial in range(4):
        qq = np.ascontiguousarray(q[rng.integers(len(q))])
        out, w = g.dense_attention(qq)
        ro, rw = _ref_attention(qq, k, v)
        assert rel_err(out, ro) < 1e-6
        assert np.max(np.abs(w - rw)) < 1e-7
        mask = np.unique(rng.integers(0, len(k), 3000)).astype(np.uint32)
        out, w = g.dense_attention(qq, mask)
        ro, rw = _ref_attention(qq, k, v, mask)
        assert rel_err(out, ro) < 1e-6
        assert np.max(np.abs(w - rw)) < 1e-7


def test_dense_oracle_validation(ctx):
    g, q, k, v = _session(ctx, 512, 1, 32, seed=43)
    with pytest.raises(cs.ParameterError, match="top-k count out of range: 0"):
        g.dense_topk(q[0], 0)
    with pytest.raises(cs.ParameterError, match="top-k count out of range"):
        g.dense_topk(q[0], 514)
    with pytest.raises(cs.ParameterError, match="mask index 513 out of range"):
        g.dense_attention(q[0], np.array([3, 513], np.uint32))
    with pytest.raises(cs.ParameterError, match="empty index set"):
        g.dense_attention(q[0], np.array([], np.uint32))


def test_recall_at_scale_matches_reference(ctx):
    """recall@K of the decode path against the dense top-K at 64K context, both
    sides: the device oracle vs the reference's dense_topk on the same rows."""
    P, d = 65536, 128
    q, k, v = workload(P, 2, d, seed=44)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=64, seed=1, score_bits=32)
    g = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, cs.RetrievalConfig(), max_decode_steps=2)
    qq = np.ascontiguousarray(q[P])
    K = cs.keep_count(0.05, P)
    truth = g.dense_topk(qq, K)
    assert np.array_equal(truth, _ref_topk(qq, np.ascontiguousarray(k[:P]), K))
    r = g.decode_step(qq, k[P], v[P])
    rec = cs.recall_at_k(r.selected, truth)
    assert 0.0 < rec <= 1.0
