"""GPU parity: the CUDA path (through the C ABI) against the reference library
(oracle/_ref) and the C restatement on identical seeded inputs.

Bar (BASELINE.json north_star): selected key-index sets identical, attention
outputs within 1e-3 relative (||o - o_ref|| / ||o_ref||, fp32 vs the
reference's fp64), tables bit-identical after every insert, counters equal.
"""
import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from oracle import bindings as ob
from tests.helpers import lockstep, random_centroids, rel_err, tables_equal, workload

pytestmark = pytest.mark.gpu
TOL = 1e-3  # relative L2 error of the attention output (north_star)


def _checker(kind):
    return ob.RefSession if (kind == "ref" and ob.ref_available()) else ob.OraSession


# ---------------- offline build ----------------

@pytest.mark.parametrize("normalize", [False, True])
def test_tables_from_centroids_bit_exact(ctx, normalize):
    P, d = 3000, 64
    q, k, v = workload(P, 1, d)
    widths = cs.uniform_widths(d, 8)
    cent = random_centroids(widths, 32, 3)
    ic = cs.IndexConfig(alpha=0.2, centroids=32, score_bits=32, normalize_keys=normalize)
    rc = cs.RetrievalConfig()
    g = cs.prefill_from_centroids(ctx, cent, k[:P], v[:P], widths, ic, rc)
    r = _checker("ref").from_centroids(cent, k[:P], v[:P], widths, ic, rc)
    assert tables_equal(g.export_index(), r.export())


def test_tables_uneven_layout_and_capacity_override(ctx):
    P, d = 700, 30
    rng = np.random.default_rng(4)
    k = rng.standard_normal((P, d)).astype(np.float32)
    k[5] = 0.0
    v = rng.standard_normal((P, d)).astype(np.float32)
    widths = cs.uniform_widths(d, 4)  # [8, 8, 7, 7]
    cent = random_centroids(widths, 5, 9)
    for ic in (cs.IndexConfig(list_capacity=700, centroids=5, score_bits=32),
               cs.IndexConfig(list_capacity=3, centroids=5, score_bits=32),
               cs.IndexConfig(alpha=1.0, centroids=5, score_bits=32)):
        g = cs.prefill_from_centroids(ctx, cent, k, v, widths, ic, cs.RetrievalConfig())
        r = _checker("ref").from_centroids(cent, k, v, widths, ic, cs.RetrievalConfig())
        assert tables_equal(g.export_index(), r.export())


@pytest.mark.parametrize("P,group,batch", [(1024, 1, 0), (4096, 1, 0), (2048, 4, 0),
                                           (1500, 2, 1000)])
def test_prefill_kmeans_bit_exact(ctx, P, group, batch):
    """GPU k-means (full-batch when n <= 4096, else mini-batch) + tables."""
    d = 128 if P == 4096 else 64
    q, k, v = workload(P, 1, d)
    widths = cs.uniform_widths(d, 8)
    qq = np.concatenate([workload(P, 1, d, dwell=dw)[0][:P]
                         for dw in (32, 16, 64, 8)[:group]])
    ic = cs.IndexConfig(alpha=0.2, centroids=64 if P == 4096 else 16, seed=1, score_bits=32,
                        batch_size=batch)
    rc = cs.RetrievalConfig()
    g = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=group)
    r = _checker("ref").prefill(qq, k[:P], v[:P], widths, ic, rc, group)
    a, b = g.export_index(), r.export()
    assert np.array_equal(a[3], b[3]), "centroids differ"
    assert tables_equal(a, b)


# ---------------- decode lockstep ----------------

DECODE_CASES = {
    "default": dict(),
    "no_passthrough": dict(rc=dict(recent_passthrough=False)),
    "period4": dict(rc=dict(search_period=4, keep_ratio=0.15)),
    "backoff": dict(rc=dict(backoff_tau=3, backoff_threshold=0.97)),
    "weights": dict(rc=dict(weights=[1.0, 2.0, 0.5, 1.0, 1.5, 1.0, 0.25, 3.0])),
    "full_keep": dict(rc=dict(keep_ratio=1.0)),
    "window_covers_budget": dict(rc=dict(keep_ratio=0.01, recent_window=64)),
    "no_window": dict(rc=dict(recent_window=0)),
    "normalize_keys": dict(ic=dict(normalize_keys=True)),
    "gqa4": dict(group=4),
}


@pytest.mark.parametrize("name", list(DECODE_CASES))
def test_decode_lockstep(ctx, name):
    case = DECODE_CASES[name]
    P, T, d = 2048, 40, 64
    q, k, v = workload(P, T, d)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=32, **case.get("ic", {}))
    rc = cs.RetrievalConfig(**case.get("rc", {}))
    grp = case.get("group", 1)
    qq = np.concatenate([q[:P]] * grp) if grp > 1 else q[:P]
    g = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=grp, max_decode_steps=T)
    r = _checker("ref").prefill(qq, k[:P], v[:P], widths, ic, rc, grp)
    assert tables_equal(g.export_index(), r.export())
    lockstep(g, r, q, k, v, P, T, group=grp, check_tables_every=10, tol=TOL)


MT_CASES = ["default", "no_passthrough", "period4", "backoff", "weights", "gqa4"]


@pytest.mark.parametrize("name", MT_CASES)
def test_decode_lockstep_multitile(ctx, name):
    """Several 4096-key select tiles per problem: split part units + merge (few
    problems), the speculative cut from step 2 on, list boundaries across tiles."""
    case = DECODE_CASES[name]
    P, T, d = 12288, 12, 64
    q, k, v = workload(P, T, d, seed=77)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=32, **case.get("ic", {}))
    rc = cs.RetrievalConfig(**case.get("rc", {}))
    grp = case.get("group", 1)
    qq = np.concatenate([q[:P]] * grp) if grp > 1 else q[:P]
    g = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=grp, max_decode_steps=T)
    r = _checker("ref").prefill(qq, k[:P], v[:P], widths, ic, rc, grp)
    lockstep(g, r, q, k, v, P, T, group=grp, check_tables_every=6, tol=TOL)


def test_c1_config_matches_reference(ctx):
    """BASELINE config 1: one head, d=128, 4K context, 95% sparsity, full defaults."""
    P, T, d = 4096, 16, 128
    q, k, v = workload(P, T, d)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=64, iterations=10, seed=1, score_bits=32)
    rc = cs.RetrievalConfig()
    g = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, rc, max_decode_steps=T)
    r = _checker("ref").prefill(q[:P], k[:P], v[:P], widths, ic, rc)
    assert g.info().list_capacity == 820
    assert tables_equal(g.export_index(), r.export())
    worst = lockstep(g, r, q, k, v, P, T, check_tables_every=8, tol=TOL)
    assert worst < 1e-5


def test_import_reference_tables_then_decode(ctx):
    """The offline -> online handoff: adopt a host CsIndex image."""
    P, T, d = 1500, 20, 32
    q, k, v = workload(P, T, d)
    widths = cs.uniform_widths(d, 4)
    ic = cs.IndexConfig(alpha=0.3, centroids=8, seed=3, score_bits=32)
    rc = cs.RetrievalConfig(keep_ratio=0.1)
    r = _checker("ref").prefill(q[:P], k[:P], v[:P], widths, ic, rc)
    lens, idx, sc, cent = r.export()
    g = cs.import_index(ctx, cent, lens, idx, sc, r.L, 0.3, k[:P], v[:P], widths, rc,
                        max_decode_steps=T)
    assert tables_equal(g.export_index(), (lens, idx, sc, cent))
    lockstep(g, r, q, k, v, P, T, check_tables_every=5)


def _import_single_list(ctx, n, cand, scores, rc):
    """One subspace, one centroid, one list = the hand-built CandidateSet of the
    reference's select_topk tests (test_retrieval.cpp:79-86)."""
    d = 4
    rng = np.random.default_rng(n)
    k = rng.standard_normal((n, d)).astype(np.float32)
    v = rng.standard_normal((n, d)).astype(np.float32)
    lens = np.array([len(cand)], np.uint32)
    order = sorted(range(len(cand)), key=lambda i: (-scores[i], cand[i]))
    idx = np.array([[cand[i] for i in order] or [0]], np.uint32)
    sc = np.array([[scores[i] for i in order] or [0.0]], np.float32)
    cent = np.array([1, 0, 0, 0], np.float32)
    return cs.import_index(ctx, cent, lens, idx, sc, max(len(cand), 1), 1.0, k, v, [4], rc,
                           max_decode_steps=1)


@pytest.mark.parametrize("cand,scores,n,rho,window,pt,want", [
    ([0, 1, 7], [9.0, 8.0, 0.1], 10, 0.5, 3, True, [0, 1, 7, 8, 9]),
    ([4], [1.0], 10, 1.0, 3, True, list(range(10))),
    ([0, 1], [9.0, 8.0], 10, 0.2, 3, True, [8, 9]),
    ([], [], 10, 0.3, 0, True, [7, 8, 9]),
    ([0, 1, 4], [5.0, 0.5, -1.0], 6, 0.5, 2, False, [0, 1, 5]),
    ([3, 5, 6, 8], [2.0, 2.0, 2.0, 2.0], 12, 0.25, 0, True, [3, 5, 6]),
    ([1, 2, 3], [-0.0, 0.0, -1.0], 8, 0.25, 0, True, [1, 2]),
])
def test_select_topk_known_answers_on_gpu(ctx, cand, scores, n, rho, window, pt, want):
    """test_retrieval.cpp:261-321 through the CUDA selection (plus tie and -0.0 cases)."""
    rc = cs.RetrievalConfig(keep_ratio=rho, recent_window=window, recent_passthrough=pt)
    s = _import_single_list(ctx, n, cand, scores, rc)
    rep = s.decode_step(np.array([1, 0, 0, 0], np.float32), np.zeros(4), np.zeros(4))
    assert rep.selected.tolist() == want


def test_select_size_property_on_gpu(ctx):
    rng = np.random.default_rng(15)
    for trial in range(25):
        n = int(1 + rng.integers(64))
        cand = [i for i in range(n) if rng.random() < 0.3]
        scores = rng.standard_normal(len(cand)).astype(np.float32).tolist()
        rc = cs.RetrievalConfig(keep_ratio=float(0.05 + 0.9 * rng.random()),
                                recent_window=int(rng.integers(8)),
                                recent_passthrough=bool(rng.random() < 0.5))
        s = _import_single_list(ctx, n, cand, scores, rc)
        rep = s.decode_step(np.array([1, 0, 0, 0], np.float32), np.zeros(4), np.zeros(4))
        ci = np.array(cand, np.uint32)
        sc = np.array(scores, np.float64)
        out = np.zeros(n, np.uint32)
        kk = ob.ora_lib().ora_select_topk(ci.ctypes.data if n and len(ci) else None,
                                          sc.ctypes.data if len(sc) else None, len(ci), n,
                                          rc.keep_ratio, rc.recent_window,
                                          int(rc.recent_passthrough), 0, out.ctypes.data)
        assert rep.selected.tolist() == out[:kk].tolist(), trial


def test_incremental_equals_batch_on_gpu(ctx):
    """test_retrieval.cpp:473-510: inserting keys one by one == building over all."""
    rng = np.random.default_rng(900)
    for seed in range(12):
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
        g = cs.prefill_from_centroids(ctx, cent, keys[:p], vals[:p], widths, ic,
                                      cs.RetrievalConfig(), max_decode_steps=extra)
        qv = rng.standard_normal(d).astype(np.float32)
        for t in range(extra):
            g.decode_step(qv, keys[p + t], vals[p + t])
        L = g.info().list_capacity
        b = cs.prefill_from_centroids(ctx, cent, keys, vals, widths,
                                      cs.IndexConfig(list_capacity=L, centroids=c, score_bits=32),
                                      cs.RetrievalConfig())
        assert tables_equal(g.export_index(), b.export_index()), seed


def test_low_buffer_refill_and_compaction(ctx):
    """Force > LOW_Q (256) evictions per table so the compaction + refill path runs."""
    P, T, d = 2048, 700, 32
    rng = np.random.default_rng(77)
    k = rng.standard_normal((P + T, d)).astype(np.float32)
    k[P:] *= 50.0  # new keys win about half of all tables every step
    v = rng.standard_normal((P + T, d)).astype(np.float32)
    q = rng.standard_normal((P + T, d)).astype(np.float32)
    widths = cs.uniform_widths(d, 2)
    cent = random_centroids(widths, 4, 5)
    ic = cs.IndexConfig(alpha=0.5, centroids=4, score_bits=32)
    rc = cs.RetrievalConfig(keep_ratio=0.02)
    g = cs.prefill_from_centroids(ctx, cent, k[:P], v[:P], widths, ic, rc, max_decode_steps=T)
    r = ob.OraSession.from_centroids(cent, k[:P], v[:P], widths, ic, rc)
    lockstep(g, r, q, k, v, P, T, check_tables_every=100)
    assert tables_equal(g.export_index(), r.export())


def test_fork_is_an_independent_copy(ctx):
    P, T, d = 1024, 12, 32
    q, k, v = workload(P, 2 * T, d)
    widths = cs.uniform_widths(d, 4)
    ic = cs.IndexConfig(alpha=0.2, centroids=8, seed=2, score_bits=32)
    rc = cs.RetrievalConfig()
    a = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, rc, max_decode_steps=2 * T)
    r = _checker("ref").prefill(q[:P], k[:P], v[:P], widths, ic, rc)
    lockstep(a, r, q, k, v, P, T)
    b = a.fork()
    # advance b on a different stream of rows; a must be unaffected
    for t in range(T):
        b.decode_step(q[P + T + t] * 0.5, k[P + T + t] * 2, v[P + T + t])
    for t in range(T, 2 * T):
        ga = a.decode_step(q[P + t], k[P + t], v[P + t])
        (sel, out, _, _), = r.step(q[P + t], k[P + t], v[P + t])
        assert np.array_equal(ga.selected, sel)
        assert rel_err(ga.output, out) < TOL
    assert tables_equal(a.export_index(), r.export())


def test_session_capacity_and_errors(ctx):
    P, d = 256, 16
    q, k, v = workload(P, 4, d)
    widths = cs.uniform_widths(d, 2)
    ic = cs.IndexConfig(alpha=0.2, centroids=4, seed=1, score_bits=32)
    with pytest.raises(cs.ParameterError, match="alpha must lie"):
        cs.prefill(ctx, q[:P], k[:P], v[:P], widths, cs.IndexConfig(alpha=0.0), cs.RetrievalConfig())
    with pytest.raises(cs.ParameterError, match="keep ratio"):
        cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, cs.RetrievalConfig(keep_ratio=0.0))
    with pytest.raises(cs.DimensionError, match="one weight per subspace"):
        cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, cs.RetrievalConfig(weights=[1.0]))
    with pytest.raises(cs.ParameterError, match="weights must be positive"):
        cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, cs.RetrievalConfig(weights=[1.0, 0.0]))
    bad = k[:P].copy()
    bad[3, 2] = np.nan
    with pytest.raises(cs.DataError, match="non-finite"):
        cs.prefill(ctx, q[:P], bad, v[:P], widths, ic, cs.RetrievalConfig())
    s = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, cs.RetrievalConfig(), max_decode_steps=2)
    s.decode_step(q[P], k[P], v[P])
    s.decode_step(q[P + 1], k[P + 1], v[P + 1])
    with pytest.raises(cs.CapacityError):
        s.decode_step(q[P + 2], k[P + 2], v[P + 2])
    with pytest.raises(cs.StreamExhaustedError, match="step 1 of 3"):
        cs.run_decode(s, q[:1], k[:1], v[:1], 3)
    with pytest.raises(cs.DataError, match="appended key"):
        s2 = s.fork(max_decode_steps=4)
        kk = k[P].copy()
        kk[0] = np.inf
        s2.decode_step(q[P], kk, v[P])


def test_c2_scale_selected_sets(ctx):
    """BASELINE config 2 shape at one KV head: 32K context, GQA group of 4 pooled."""
    P, T, d = 32768, 3, 128
    widths = cs.uniform_widths(d, 8)
    qs = [workload(P, T, d, dwell=dw) for dw in (32, 16, 64, 8)]
    k, v = qs[0][1], qs[0][2]
    qq = np.concatenate([x[0][:P] for x in qs])
    ic = cs.IndexConfig(alpha=0.2, centroids=64, seed=1, score_bits=32)
    rc = cs.RetrievalConfig()
    g = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=4, max_decode_steps=T)
    r = _checker("ref").prefill(qq, k[:P], v[:P], widths, ic, rc, 4)
    assert tables_equal(g.export_index(), r.export())
    qstep = np.stack([np.stack([x[0][P + t] for x in qs]) for t in range(T)])
    lockstep(g, r, qstep, k, v, P, T, group=4)


@pytest.mark.parametrize("ctas", ["", "1"])
def test_union_attend_fork_batch(ctx, monkeypatch, ctas):
    """Batch decode of forks that share one prefill (config c3's shape): the
    union attend path (attend_union.cu, CSATTN_UNION=1) must give every
    (sequence, head) the same selected set and output as decoding that fork
    alone. 20 forks x GQA 4 = 80 problems on one prefill -> two union groups of
    40; a second prefill with 2 forks (8 problems) in the same batch stays on
    the per-problem path. ctas="1": every work item on one persistent CTA."""
    monkeypatch.setenv("CSATTN_UNION", "1")
    if ctas:
        monkeypatch.setenv("CSATTN_UNION_CTAS", ctas)
    P, T, d, F = 8192, 5, 128, 20
    q, k, v = workload(P, 64, d, seed=31)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=32, seed=1, score_bits=32)
    rc = cs.RetrievalConfig()
    qq = np.concatenate([q[:P]] * 4)
    base = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=4, max_decode_steps=T)
    q2, k2, v2 = workload(4096, 8, d, seed=32)
    base2 = cs.prefill(ctx, np.concatenate([q2[:4096]] * 4), k2[:4096], v2[:4096], widths, ic, rc,
                       group=4, max_decode_steps=T)
    batch = [base.fork() for _ in range(F)] + [base2.fork() for _ in range(2)]
    alone = [base.fork() for _ in range(F)] + [base2.fork() for _ in range(2)]
    rng = np.random.default_rng(5)
    worst = 0.0
    for t in range(T):
        # fork f queries with prefill rows near its own offset; its own appended rows
        Q = np.stack([q[(P + 3 * f + t + 8 * h) % (P + 64)] for f in range(F) for h in range(4)] +
                     [q2[4096 + t]] * 8).astype(np.float32)
        Q *= (1.0 + 0.1 * rng.standard_normal((len(Q), 1))).astype(np.float32)
        Kn = np.stack([k[P + (f + t) % 64] for f in range(F)] + [k2[4096 + t]] * 2)
        Vn = np.stack([v[P + (f + 2 * t) % 64] for f in range(F)] + [v2[4096 + t]] * 2)
        out, sel = cs.decode_batch(batch, Q, Kn, Vn)
        for f, s in enumerate(alone):
            reps = s.decode_step(Q[4 * f:4 * f + 4], Kn[f], Vn[f])
            for h, r in enumerate(reps):
                row = 4 * f + h
                assert np.array_equal(sel[row, :r.k], r.selected), (t, f, h)
                worst = max(worst, rel_err(out[row], r.output))
    assert worst < 1e-4, worst


@pytest.mark.parametrize("gr", ["4", "8"])
@pytest.mark.parametrize("group", [1, 4])
def test_attend128_no_weights_path(ctx, monkeypatch, gr, group):
    """attend128 (d = 128) as decode_batch runs it: no weights, prefill-only
    batches on the specialised loop, batches holding appended rows (the recent
    window keeps them selected) on the mixed loop. Both row-group sizes.
    Selected sets exact, outputs within 1e-3 of the reference."""
    monkeypatch.setenv("CSATTN_ATT_GR", gr)
    P, T, d = 4096, 24, 128
    q, k, v = workload(P, T, d, seed=81)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=32, seed=1, score_bits=32)
    rc = cs.RetrievalConfig(keep_ratio=0.1)
    qq = np.concatenate([q[:P]] * group) if group > 1 else q[:P]
    g = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=group, max_decode_steps=T)
    r = _checker("ref").prefill(qq, k[:P], v[:P], widths, ic, rc, group)
    worst = 0.0
    for t in range(T):
        Q = np.stack([q[P + t] * (1 + 0.05 * h) for h in range(group)]).astype(np.float32)
        out, sel = cs.decode_batch([g], Q, k[P + t][None], v[P + t][None])
        for h, (rs, ro, _, _) in enumerate(r.step(Q, k[P + t], v[P + t])):
            assert np.array_equal(sel[h, :len(rs)], rs), (t, h)
            if t > 0:
                assert (rs >= P).any()  # appended rows are in the set: mixed batches run
            worst = max(worst, rel_err(out[h], ro))
    assert worst <= 1e-3, worst


def test_prefill_batch_equals_single_prefills(ctx):
    """csattn_prefill_batch (one k-means launch for a layer's KV heads, per-head
    seeds) builds exactly the sessions n single prefills build: centroids and
    tables bit-identical, and the first decode step selects the same keys."""
    P, d, grp = 3072, 64, 2
    widths = cs.uniform_widths(d, 8)
    rc = cs.RetrievalConfig()
    rows, ics = [], []
    for h in range(3):
        q, k, v = workload(P, 2, d, seed=90 + h)
        rows.append((np.concatenate([q[:P]] * grp), k[:P], v[:P]))
        ics.append(cs.IndexConfig(alpha=0.2, centroids=16, seed=7 + h, score_bits=32))
    batch = cs.prefill_batch(ctx, rows, widths, ics, rc, group=grp, max_decode_steps=2)
    for (qq, k, v), ic, b in zip(rows, ics, batch):
        single = cs.prefill(ctx, qq, k, v, widths, ic, rc, group=grp, max_decode_steps=2)
        ea, eb = b.export_index(), single.export_index()
        assert np.array_equal(ea[3], eb[3]), "centroids differ"
        assert tables_equal(ea, eb)
        Q = np.stack([qq[5], qq[P + 9]]).astype(np.float32)
        ra = b.decode_step(Q, k[1], v[1])
        rb = single.decode_step(Q, k[1], v[1])
        for x, y in zip(ra, rb):
            assert np.array_equal(x.selected, y.selected)
    # an all-zero training set in one entry refuses the whole batch
    bad = [rows[0], (np.zeros_like(rows[1][0]), rows[1][1], rows[1][2])]
    with pytest.raises(cs.DataError):
        cs.prefill_batch(ctx, bad, widths, ics[:2], rc, group=grp)


@pytest.mark.parametrize("rows", ["128", "256", "512"])
def test_attend_chunk_rows(ctx, monkeypatch, rows):
    """Attention chunking by 128, 256 or 512 rows per CTA (chosen by launch
    size: c2 128, c4 256, c3 512): same selected sets as the reference, outputs within
    1e-3, for d = 128 (attend128) and d = 64 (generic kernel)."""
    monkeypatch.setenv("CSATTN_ATT_ROWS", rows)
    for d, P in ((128, 8192), (64, 4096)):
        T = 6
        q, k, v = workload(P, T, d, seed=83)
        widths = cs.uniform_widths(d, 8)
        ic = cs.IndexConfig(alpha=0.2, centroids=32, seed=1, score_bits=32)
        rc = cs.RetrievalConfig(keep_ratio=0.2)  # K = 1639 / 820: several chunks
        qq = np.concatenate([q[:P]] * 4)
        g = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=4, max_decode_steps=T)
        r = _checker("ref").prefill(qq, k[:P], v[:P], widths, ic, rc, 4)
        worst = 0.0
        for t in range(T):
            Q = np.stack([q[P + t] * (1 + 0.05 * h) for h in range(4)]).astype(np.float32)
            out, sel = cs.decode_batch([g], Q, k[P + t][None], v[P + t][None])
            for h, (rs, ro, _, _) in enumerate(r.step(Q, k[P + t], v[P + t])):
                assert np.array_equal(sel[h, :len(rs)], rs), (d, t, h)
                worst = max(worst, rel_err(out[h], ro))
        assert worst <= 1e-3, (d, worst)
