"""CPU: pin the C restatement (oracle/csattn_oracle.c) against the reference's
own known answers (proj/tests/*.cpp) and against the reference library itself
(oracle/_ref, built from the unmodified sources)."""
import ctypes as C
import math

import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from oracle import bindings as ob
from tests.helpers import random_centroids, tables_equal, workload

ora = ob.ora_lib()


def f32p(a):
    return a.ctypes.data


# ---------------- known answers from the reference test suite ----------------

def test_ceil_ratio_known_answers():  # test_core.cpp:260-266
    for r, n, want in [(0.05, 7936, 397), (0.05, 8000, 400), (0.2, 1000, 200),
                       (0.15, 8192, 1229), (1.0, 123, 123), (0.5, 3, 2)]:
        assert ora.ora_ceil_ratio(r, n) == want


def test_keep_count_known_answers():  # test_retrieval.cpp:123-132
    out = C.c_uint64()
    for rho, n, want in [(0.05, 10, 1), (0.05, 1, 1), (0.05, 8192, 410), (1.0, 77, 77),
                         (0.5, 3, 2)]:
        assert ora.ora_keep_count(rho, n, C.byref(out)) == 0
        assert out.value == want
    assert ora.ora_keep_count(0.0, 10, C.byref(out)) == 3  # ParameterError
    assert ora.ora_keep_count(1.5, 10, C.byref(out)) == 3


def test_score_keys_known_answers():  # test_index.cpp:128-147
    keys = np.array([2, 1, 0, 3, -1, 4], np.float32)
    c = np.array([1, 0], np.float32)
    out = np.zeros(3, np.float32)
    ora.ora_score_keys(f32p(c), f32p(keys), 3, 2, 0, 2, 0, f32p(out))
    assert out.tolist() == [2.0, 0.0, -1.0]
    ora.ora_score_keys(f32p(c), f32p(keys), 3, 2, 0, 2, 1, f32p(out))
    assert out[0] == pytest.approx(2 / math.sqrt(5), rel=1e-6)
    assert out[1] == 0.0
    assert out[2] == pytest.approx(-1 / math.sqrt(17), rel=1e-6)
    zk = np.zeros(6, np.float32)
    ora.ora_score_keys(f32p(c), f32p(zk), 3, 2, 0, 2, 1, f32p(out))
    assert out.tolist() == [0.0, 0.0, 0.0]


def test_two_key_attention_closed_form():  # test_core.cpp:96-112
    keys = np.array([1, 0, 0, 1], np.float32)
    q = np.array([1, 0], np.float32)
    out = np.zeros(2, np.float32)
    w = np.zeros(2, np.float32)
    ora.ora_attention(f32p(q), f32p(keys), f32p(keys), 2, 2, None, 0, f32p(out), f32p(w))
    assert w[0] == pytest.approx(0.669761549326656925616794945834, rel=1e-6)
    assert w[1] == pytest.approx(0.330238450673343074383205054166, rel=1e-6)
    assert out[0] == pytest.approx(w[0])


def _select(cidx, cscore, n, rho, window, passthrough=True):
    ci = np.array(cidx, np.uint32)
    sc = np.array(cscore, np.float64)
    out = np.zeros(n, np.uint32)
    k = ora.ora_select_topk(ci.ctypes.data if len(ci) else None,
                            sc.ctypes.data if len(sc) else None, len(ci), n, rho, window,
                            int(passthrough), 0, out.ctypes.data)
    return out[:k].tolist()


def test_select_topk_known_answers():  # test_retrieval.cpp:261-321
    assert _select([0, 1, 7], [9.0, 8.0, 0.1], 10, 0.5, 3) == [0, 1, 7, 8, 9]
    assert _select([4], [1.0], 10, 1.0, 3) == list(range(10))
    assert _select([0, 1], [9.0, 8.0], 10, 0.2, 3) == [8, 9]
    assert _select([], [], 10, 0.3, 0) == [7, 8, 9]
    assert _select([0, 1, 4], [5.0, 0.5, -1.0], 6, 0.5, 2, passthrough=False) == [0, 1, 5]
    rng = np.random.default_rng(12)
    sc = rng.standard_normal(200)
    got = _select(list(range(200)), sc.tolist(), 200, 0.05, 0)
    order = sorted(range(200), key=lambda i: (-sc[i], i))[:10]
    assert got == sorted(order)


def test_select_topk_size_property():  # test_retrieval.cpp:323-345
    rng = np.random.default_rng(15)
    for _ in range(40):
        n = int(1 + rng.integers(64))
        idx = [i for i in range(n) if rng.random() < 0.3]
        sc = rng.standard_normal(len(idx)).tolist()
        rho = 0.05 + 0.9 * rng.random()
        got = _select(idx, sc, n, rho, int(rng.integers(8)), bool(rng.random() < 0.5))
        assert len(got) == max(1, math.ceil(rho * n - 1e-9))
        assert got == sorted(set(got)) and all(i < n for i in got)


# ---------------- restatement == reference library ----------------

@pytest.mark.usefixtures("ref_ok")
def test_synthetic_generator_matches_reference():
    spec = cs.SyntheticSpec(rows=300, dim=64, clusters=8, seed=2026)
    a = cs.make_synthetic(spec)
    b = ob.ref_make_synthetic(spec)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    # prefix stability (synthetic.hpp:38-41)
    spec2 = cs.SyntheticSpec(rows=100, dim=64, clusters=8, seed=2026)
    c = cs.make_synthetic(spec2)
    assert np.array_equal(c[1], a[1][:100])


CASES = {
    "default": dict(),
    "no_passthrough": dict(rc=dict(recent_passthrough=False)),
    "period4": dict(rc=dict(search_period=4, keep_ratio=0.15)),
    "backoff": dict(rc=dict(backoff_tau=3, backoff_threshold=0.97)),
    "weights": dict(rc=dict(weights=[1.0, 2.0, 0.5, 1.0, 1.5, 1.0, 0.25, 3.0])),
    "full_keep": dict(rc=dict(keep_ratio=1.0)),
    "normalize_keys": dict(ic=dict(normalize_keys=True)),
    "gqa4": dict(group=4),
}


@pytest.mark.usefixtures("ref_ok")
@pytest.mark.parametrize("name", list(CASES))
def test_restatement_matches_reference(name):
    case = CASES[name]
    P, T, d = 1024, 24, 64
    q, k, v = workload(P, T, d)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=32, **case.get("ic", {}))
    rc = cs.RetrievalConfig(**case.get("rc", {}))
    g = case.get("group", 1)
    qq = np.concatenate([q[:P]] * g) if g > 1 else q[:P]
    R = ob.RefSession.prefill(qq, k[:P], v[:P], widths, ic, rc, g)
    O = ob.OraSession.prefill(qq, k[:P], v[:P], widths, ic, rc, g)
    assert tables_equal(R.export(), O.export())
    for t in range(T):
        qs = np.stack([q[P + t]] * g)
        for (s1, o1, w1, r1), (s2, o2, w2, r2) in zip(R.step(qs, k[P + t], v[P + t]),
                                                      O.step(qs, k[P + t], v[P + t])):
            assert np.array_equal(s1, s2)
            assert np.array_equal(o1, o2)
            assert np.array_equal(w1, w2)
            for f in ("k", "searched", "centroid_dot_ops", "gathered_entries", "reduce_ops",
                      "inserts_applied", "inserts_attempted", "insert_dot_ops"):
                assert getattr(r1, f) == getattr(r2, f), f
    assert tables_equal(R.export(), O.export())


@pytest.mark.usefixtures("ref_ok")
def test_restatement_kmeans_full_and_minibatch():
    rng = np.random.default_rng(5)
    for n, batch in [(900, 0), (6000, 0), (3000, 1000)]:
        pts = rng.standard_normal((n, 16)).astype(np.float32)
        pts[7] = 0.0  # a degenerate row is dropped
        out = np.zeros(64 * 16, np.float32)
        # reference through build_index_from a 1-subspace layout
        ic = cs.IndexConfig(alpha=1.0, centroids=64, seed=0, batch_size=batch, score_bits=32)
        # build_index uses mix_seed(seed, 0) for subspace 0
        seed0 = ob.ref_lib().csref_mix_seed(0, 0)
        out2 = np.zeros_like(out)
        assert ora.ora_cosine_kmeans(pts.ctypes.data, n, 16, 64, 10, batch, seed0, 1e-7,
                                     out2.ctypes.data) == 0
        R = ob.RefSession.prefill(pts, pts, pts, [16], ic, cs.RetrievalConfig())
        assert np.array_equal(R.export()[3], out2)


@pytest.mark.usefixtures("ref_ok")
def test_restatement_incremental_equals_batch():  # test_retrieval.cpp:473-510 (oracle side)
    rng = np.random.default_rng(900)
    for seed in range(10):
        d = int(4 * (1 + rng.integers(3)))
        m = int(1 + rng.integers(min(4, d)))
        c = int(1 + rng.integers(6))
        p = int(16 + rng.integers(113))
        extra = int(1 + rng.integers(128))
        alpha = float(0.1 + 0.9 * rng.random())
        widths = cs.uniform_widths(d, m)
        keys = rng.standard_normal((p + extra, d)).astype(np.float32)
        vals = rng.standard_normal((p + extra, d)).astype(np.float32)
        cent = random_centroids(widths, c, seed)
        ic = cs.IndexConfig(alpha=alpha, centroids=c, score_bits=32)
        O = ob.OraSession.from_centroids(cent, keys[:p], vals[:p], widths, ic,
                                         cs.RetrievalConfig())
        R = ob.RefSession.from_centroids(cent, keys[:p], vals[:p], widths, ic,
                                         cs.RetrievalConfig())
        q = rng.standard_normal(d).astype(np.float32)
        for t in range(extra):
            O.step(q, keys[p + t], vals[p + t])
            R.step(q, keys[p + t], vals[p + t])
        assert tables_equal(O.export(), R.export())
