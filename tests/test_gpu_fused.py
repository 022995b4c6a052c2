"""The fused cluster step (csrc/fused.cu: a problem's routing, gather /
accumulate, top-K selection and attention in one thread-block cluster, for
small batches) against the reference library, step by step: identical
selected sets, bit-identical candidate sets, outputs within 1e-3, counters,
tables after the inserts. Both cluster shapes (8 CTAs of up to 14 x 512 keys,
N <= 57344; 16 CTAs of up to 32 x 512 keys, N <= 262144) and every retrieval
mode (passthrough or not, backoff, weights, schedules with the cached
candidate scores, GQA). CSATTN_FUSED=1 forces it; =0 keeps the multi-kernel
path for the same cases."""
import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from oracle import bindings as ob
from tests.helpers import lockstep, tables_equal, workload

pytestmark = pytest.mark.gpu

CASES = {
    "default": {},
    "no_passthrough": dict(rc=dict(recent_passthrough=False)),
    "period4": dict(rc=dict(search_period=4, keep_ratio=0.15)),
    "backoff": dict(rc=dict(backoff_tau=3, backoff_threshold=0.97)),
    "weights": dict(rc=dict(weights=[1.0, 2.0, 0.5, 1.0, 1.5, 1.0, 0.25, 3.0])),
    "full_keep": dict(rc=dict(keep_ratio=1.0)),
    "window_covers_budget": dict(rc=dict(keep_ratio=0.01, recent_window=64)),
    "no_window": dict(rc=dict(recent_window=0)),
    "gqa4": dict(group=4),
}


def _run(monkeypatch, mode, P, T, d, name, seed=5):
    monkeypatch.setenv("CSATTN_FUSED", str(mode))
    ctx = cs.Context(0)  # reads CSATTN_FUSED
    case = CASES[name]
    q, k, v = workload(P, T, d, seed=seed)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=32, **case.get("ic", {}))
    rc = cs.RetrievalConfig(**case.get("rc", {}))
    grp = case.get("group", 1)
    qq = np.concatenate([q[:P]] * grp) if grp > 1 else q[:P]
    g = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=grp, max_decode_steps=T)
    r = ob.RefSession.prefill(qq, k[:P], v[:P], widths, ic, rc, grp)
    assert tables_equal(g.export_index(), r.export())
    launches0 = ctx.launches
    lockstep(g, r, q, k, v, P, T, group=grp, check_tables_every=max(1, T // 2), want_weights=False)
    return ctx.launches - launches0


@pytest.fixture(autouse=True)
def _needs_ref():
    if not ob.ref_available():
        pytest.skip("oracle/_ref not built")


@pytest.mark.parametrize("name", list(CASES))
def test_fused_cluster8_matches_reference(monkeypatch, name):
    """8-CTA clusters (N = 12288: 3 x 512 keys per CTA)."""
    n = _run(monkeypatch, 1, 12288, 10, 128, name)
    assert n == 2 * 10  # fused step + insert per decode step


@pytest.mark.parametrize("P,name", [(40000, "default"), (40000, "no_passthrough"), (40000, "gqa4"),
                                    (70000, "default"), (70000, "period4"), (100000, "backoff"),
                                    (131072, "default")])
def test_fused_larger_contexts_match_reference(monkeypatch, P, name):
    """N = 40000 (8 CTAs x 10 ranges), 70000 .. 131072 + steps (16-CTA clusters,
    9 .. 17 ranges per CTA: the c4 shape)."""
    _run(monkeypatch, 1, P, 5, 128, name, seed=9)


@pytest.mark.parametrize("name", ["default", "no_passthrough", "period4", "gqa4"])
def test_multikernel_path_without_weights(monkeypatch, name):
    """The same small cases through the multi-kernel path (CSATTN_FUSED=0)."""
    n = _run(monkeypatch, 0, 12288, 8, 128, name)
    assert n > 2 * 8


def test_fused_threshold_bin_overflow(monkeypatch):
    """Many equal scores (duplicated keys): the threshold bin exceeds the
    bucket and CTA 0 ranks over the whole cluster (radix passes)."""
    monkeypatch.setenv("CSATTN_FUSED", "1")
    ctx = cs.Context(0)
    P, T, d = 20000, 3, 128
    q, k, v = workload(P, T, d, seed=3)
    k[:P] = k[0]  # every prefill key identical: all sums tie per list pattern
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.5, centroids=4, seed=1, score_bits=32)
    rc = cs.RetrievalConfig(keep_ratio=0.3)
    g = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, rc, max_decode_steps=T)
    r = ob.RefSession.prefill(q[:P], k[:P], v[:P], widths, ic, rc, 1)
    lockstep(g, r, q, k, v, P, T, want_weights=False)


def _pdl_batch(monkeypatch, pdl, P, T, nf):
    monkeypatch.setenv("CSATTN_FUSED", "1")
    monkeypatch.setenv("CSATTN_PDL", str(pdl))
    ctx = cs.Context(0)  # reads CSATTN_FUSED / CSATTN_PDL
    d, grp = 128, 4
    q, k, v = workload(P, T + nf, d, seed=13)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.05, centroids=16, seed=1, score_bits=32)  # small L: many evictions
    qq = np.concatenate([q[:P]] * grp)
    base = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, cs.RetrievalConfig(), group=grp,
                      max_decode_steps=T)
    forks = [base.fork(T) for _ in range(nf)]
    outs, sels = [], []
    for t in range(T):
        Q = np.stack([q[P + f + t] for f in range(nf) for _ in range(grp)])
        out, sel = cs.decode_batch(forks, Q, k[P + t:P + t + nf], v[P + t:P + t + nf])
        outs.append(out.copy())
        sels.append(sel.copy())
    return outs, sels, [f.export_index() for f in forks]


def test_insert_programmatic_dependent_of_fused_step(monkeypatch):
    """The insert after the fused step is a programmatic dependent (it scores the
    key and reads table state while the fused kernel runs, and writes the tables
    after griddepcontrol.wait): outputs, selected sets and the tables after every
    step's inserts are bit-identical to the serialised launch (CSATTN_PDL=0), over
    a c2-like batch (8 sessions x GQA 4) with frequent evictions."""
    a = _pdl_batch(monkeypatch, 4, 20000, 12, 8)
    b = _pdl_batch(monkeypatch, 0, 20000, 12, 8)
    for oa, ob_ in zip(a[0], b[0]):
        assert np.array_equal(oa, ob_)
    for sa, sb in zip(a[1], b[1]):
        assert np.array_equal(sa, sb)
    for ta, tb in zip(a[2], b[2]):
        assert tables_equal(ta, tb)
