"""Exactness and error-contract hardening on the GPU path (VERDICT r1 "exactness
hardening"):
  * a -0.0f table score is a PRESENT key scored +0.0 (reduce_by_key starts its
    sums at 0.0, retrieval.cpp:111-148; float() of a tiny negative dot is -0.0f,
    index.cpp:81 / retrieval.cpp:293-294), also after a CSAT export round trip;
  * a non-finite appended row on the DEVICE-pointer path raises DataError like
    KvStore::append (core.cpp:71-79) and leaves the KV rows and tables as they
    were; found only after later steps were queued, the session refuses further
    work;
  * one session twice in a batch is refused;
  * raising search_period mid-session reuses the last search's candidates
    exactly as decode_search does (retrieval.cpp:237-238), or is refused when
    they were not kept.
"""
import ctypes as C

import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from paper_2604_08584_b200 import _abi
from oracle import bindings as ob
from tests.helpers import lockstep, rel_err, tables_equal, workload

pytestmark = pytest.mark.gpu


def _single_list(ctx, n, cand, scores, rc):
    d = 4
    rng = np.random.default_rng(n)
    k = rng.standard_normal((n, d)).astype(np.float32)
    v = rng.standard_normal((n, d)).astype(np.float32)
    lens = np.array([len(cand)], np.uint32)
    order = sorted(range(len(cand)), key=lambda i: (-scores[i], cand[i]))
    idx = np.array([[cand[i] for i in order]], np.uint32)
    sc = np.array([[scores[i] for i in order]], np.float32)
    cent = np.array([1, 0, 0, 0], np.float32)
    g = cs.import_index(ctx, cent, lens, idx, sc, len(cand), 1.0, k, v, [4], rc, max_decode_steps=2)
    r = ob.RefSession.from_index(cent, lens, idx, sc, len(cand), 1.0, k, v, [4], rc)
    return g, r, k, v


@pytest.mark.parametrize("pt", [True, False])
def test_negative_zero_table_score_is_a_present_key(ctx, ref_ok, pt):
    # key 1 carries -0.0f: present at +0.0, so with K = 2 the set is {1, 5};
    # dropping it as "not gathered" would pad with the newest key 7 instead
    rc = cs.RetrievalConfig(keep_ratio=0.25, recent_window=0, recent_passthrough=pt)
    g, r, k, v = _single_list(ctx, 8, [1, 5], [-0.0, -1.0], rc)
    # the stored bits survive the import (export is byte-identical)
    lens, idx, sc, _ = g.export_index()
    assert sc[0, :2].view(np.uint32).tolist() == [0x80000000, np.float32(-1.0).view(np.uint32)]
    g.keep_candidates(True)
    q = np.array([1, 0, 0, 0], np.float32)
    rep = g.decode_step(q, k[0], v[0])
    (sel, out, _, _), = r.step(q, k[0], v[0])
    assert rep.selected.tolist() == sel.tolist() == [1, 5]
    assert rel_err(rep.output, out) <= 1e-6
    ci, cv = g.candidates(0)
    ri, rv = r.candidates(0)
    assert ci.tolist() == ri.tolist() == [1, 5]
    assert cv.view(np.uint64).tolist() == rv.view(np.uint64).tolist()
    assert cv[0] == 0.0 and not np.signbit(cv[0])  # +0.0, as 0.0 + (-0.0)
    assert tables_equal(g.export_index(), r.export())
    # CSAT image: the -0.0 score bits round-trip as the reference writes them
    assert g.serialize() == r.serialize(32)


def test_negative_zero_scores_from_inserts(ctx, ref_ok):
    """Inserted keys whose centroid dot is a tiny negative number (below 2^-150
    in magnitude) get -0.0f table scores (retrieval.cpp:293-294). With rho = 0.6
    those zero-score keys are selected when present: lockstep against the
    reference (candidate sets bit-exact, selected sets, tables)."""
    P, T, d = 512, 24, 8
    rng = np.random.default_rng(3)
    k = rng.standard_normal((P + T, d)).astype(np.float32)
    v = rng.standard_normal((P + T, d)).astype(np.float32)
    q = (0.01 * rng.standard_normal((P + T, d))).astype(np.float32)
    q[:, 1] += 1.0
    q[:, 5] += 1.0  # routes to centroid 0 of both subspaces
    sub = np.array([[1e-10, 1, 0, 0], [1, 0, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1]], np.float32)
    cent = np.concatenate([sub.reshape(-1)] * 2)
    for t in range(0, T, 2):  # dot with centroid 0: 1e-10 * -1e-40 -> float -0.0
        k[P + t] = 0.0
        k[P + t, 0] = np.float32(-1e-40)
        k[P + t, 4] = np.float32(-1e-40)
    ic = cs.IndexConfig(alpha=0.9, centroids=4, score_bits=32)
    rc = cs.RetrievalConfig(keep_ratio=0.6, recent_window=0)
    g = cs.prefill_from_centroids(ctx, cent, k[:P], v[:P], [4, 4], ic, rc, max_decode_steps=T)
    r = ob.RefSession.from_centroids(cent, k[:P], v[:P], [4, 4], ic, rc)
    lockstep(g, r, q, k, v, P, T, check_tables_every=4)
    sc = g.export_index()[2]
    assert (sc.view(np.uint32) == 0x80000000).any(), "no -0.0f table score was produced"


def _torch():
    torch = pytest.importorskip("torch")
    return torch


def test_device_path_nonfinite_append_raises_and_rolls_back(ctx, ref_ok):
    torch = _torch()
    P, T, d = 1024, 6, 32
    q, k, v = workload(P, T, d)
    widths = cs.uniform_widths(d, 4)
    ic = cs.IndexConfig(alpha=0.2, centroids=8, seed=1, score_bits=32)
    rc = cs.RetrievalConfig()
    a = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, rc, max_decode_steps=T)
    b = a.fork(T)
    r = ob.RefSession.prefill(q[:P], k[:P], v[:P], widths, ic, rc)
    lib = cs.lib()
    hs = (C.c_void_p * 2)(a.h.value, b.h.value)

    def step(qrows, krows, vrows, flags=0):
        qd = torch.from_numpy(np.ascontiguousarray(qrows)).cuda()
        kd = torch.from_numpy(np.ascontiguousarray(krows)).cuda()
        vd = torch.from_numpy(np.ascontiguousarray(vrows)).cuda()
        od = torch.empty((2, d), dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        st = lib.csattn_decode_batch(ctx.h, 2, hs, C.c_void_p(qd.data_ptr()), C.c_void_p(kd.data_ptr()),
                                     C.c_void_p(vd.data_ptr()), C.c_void_p(od.data_ptr()), None, 0, flags)
        cs._check(st)
        return od.cpu().numpy()

    bad_k = np.stack([k[P], k[P]])
    bad_k[1, 3] = np.nan  # session b's key is non-finite
    tab_b = b.export_index()
    with pytest.raises(cs.DataError, match="appended key contains a non-finite value"):
        step(np.stack([q[P], q[P]]), bad_k, np.stack([v[P], v[P]]))
    # a appended its row; b kept its store and tables and its context length
    assert a.context_len == P + 1 and b.context_len == P
    assert tables_equal(b.export_index(), tab_b)
    (sel, out, _, _), = r.step(q[P], k[P], v[P])
    # the value path too
    bad_v = np.stack([v[P + 1], v[P + 1]])
    bad_v[0, 0] = np.inf
    with pytest.raises(cs.DataError, match="appended value contains a non-finite value"):
        step(np.stack([q[P + 1], q[P + 1]]), np.stack([k[P + 1], k[P]]), bad_v)
    assert a.context_len == P + 1
    # a continues exactly like the reference
    (sel, out, _, _), = r.step(q[P + 1], k[P + 1], v[P + 1])
    ga = a.decode_step(q[P + 1], k[P + 1], v[P + 1])
    assert np.array_equal(ga.selected, sel) and rel_err(ga.output, out) <= 1e-3
    assert tables_equal(a.export_index(), r.export())
    # found only after a later unsynchronised step was queued: refused from then on
    c = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, rc, max_decode_steps=T)
    hs1 = (C.c_void_p * 1)(c.h.value)
    kd = torch.from_numpy(np.where(np.arange(d) == 0, np.nan, k[P]).astype(np.float32)[None]).cuda()
    qd = torch.from_numpy(q[P][None].copy()).cuda()
    vd = torch.from_numpy(v[P][None].copy()).cuda()
    od = torch.empty((1, d), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    cs._check(lib.csattn_decode_batch(ctx.h, 1, hs1, C.c_void_p(qd.data_ptr()), C.c_void_p(kd.data_ptr()),
                                      C.c_void_p(vd.data_ptr()), C.c_void_p(od.data_ptr()), None, 0,
                                      _abi.NO_SYNC))
    ctx.synchronize()
    with pytest.raises(cs.DataError, match="unusable"):
        c.decode_step(q[P + 1], k[P + 1], v[P + 1])


def test_duplicate_session_in_batch_is_refused(ctx):
    P, d = 256, 16
    q, k, v = workload(P, 2, d)
    s = cs.prefill(ctx, q[:P], k[:P], v[:P], cs.uniform_widths(d, 2),
                   cs.IndexConfig(alpha=0.2, centroids=4, seed=1, score_bits=32), cs.RetrievalConfig(),
                   max_decode_steps=2)
    with pytest.raises(cs.ParameterError, match="appears twice"):
        cs.decode_batch([s, s], np.stack([q[P], q[P]]), np.stack([k[P], k[P]]), np.stack([v[P], v[P]]))
    assert s.context_len == P


def test_raising_search_period_mid_session(ctx, ref_ok):
    P, T, d = 2048, 16, 64
    q, k, v = workload(P, T, d)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=32)
    rc1 = cs.RetrievalConfig(keep_ratio=0.1)
    rc4 = cs.RetrievalConfig(keep_ratio=0.1, search_period=4)
    # without kept candidates the switch is refused (the last search's set is gone)
    g0 = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, rc1, max_decode_steps=T)
    g0.decode_step(q[P], k[P], v[P])
    with pytest.raises(cs.ParameterError, match="keep_candidates"):
        g0.set_retrieval(rc4)
    # with them: decode_search's reuse of state.cached, step for step
    g = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, rc1, max_decode_steps=T)
    g.keep_candidates(True)
    r = ob.RefSession.prefill(q[:P], k[:P], v[:P], widths, ic, rc1)
    for t in range(T):
        if t == 5:  # step 5: 5 % 4 != 0 -> the reference reuses step 4's candidates
            g.set_retrieval(rc4)
            r.set_retrieval(rc4)
        rep = g.decode_step(q[P + t], k[P + t], v[P + t])
        (sel, out, _, rr), = r.step(q[P + t], k[P + t], v[P + t])
        assert rep.searched == bool(rr.searched), t
        assert np.array_equal(rep.selected, sel), t
        assert rel_err(rep.output, out) <= 1e-3, t
    assert tables_equal(g.export_index(), r.export())
