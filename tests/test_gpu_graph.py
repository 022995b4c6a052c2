"""run_decode as one CUDA graph (csattn_decode_run).
T steps of a session set captured and launched once must equal T calls of
decode_batch step for step (bit-identical selections and outputs, same table
state afterwards), follow the reference under period reuse and k overrides,
and leave the sessions untouched when it refuses."""
import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from oracle import bindings as ob
from tests.helpers import rel_err, tables_equal, workload

pytestmark = pytest.mark.gpu


def _setup(ctx, P, d, T, group, rc, forks, seed):
    q, k, v = workload(P, T + 8, d, seed=seed)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=32, seed=1, score_bits=32)
    qq = np.concatenate([q[:P]] * group) if group > 1 else q[:P]
    base = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=group, max_decode_steps=2 * T)
    return q, k, v, base, [base.fork() for _ in range(forks)], [base.fork() for _ in range(forks)]


def _inputs(q, k, v, P, T, F, group):
    Q = np.stack([np.stack([q[P + t] * (1 + 0.1 * f) for f in range(F) for _ in range(group)])
                  for t in range(T)]).astype(np.float32)
    K = np.stack([np.stack([k[P + (t + f) % (T + 8)] for f in range(F)]) for t in range(T)])
    V = np.stack([np.stack([v[P + (t + 2 * f) % (T + 8)] for f in range(F)]) for t in range(T)])
    return Q, K, V


@pytest.mark.parametrize("group,schedule", [(1, "0.05-step-1"), (4, "0.15-step-4")])
def test_graph_run_equals_batch_steps(ctx, group, schedule):
    P, d, T, F = 8192, 128, 12, 3
    rho, per = cs.parse_schedule(schedule)
    rc = cs.RetrievalConfig(keep_ratio=rho, search_period=per)
    q, k, v, base, gs, bs = _setup(ctx, P, d, T, group, rc, F, seed=71)
    Q, K, V = _inputs(q, k, v, P, T, F, group)
    go, gsel = cs.decode_run(gs, Q, K, V)
    for t in range(T):
        bo, bsel = cs.decode_batch(bs, Q[t], K[t], V[t])
        kk = cs.keep_count(rho, P + t)
        assert np.array_equal(gsel[t, :, :kk], bsel[:, :kk]), t
        assert np.array_equal(go[t], bo), t
    for a, b in zip(gs, bs):
        assert a.serialize() == b.serialize()
        assert a.context_len == b.context_len == P + T
    # the sessions keep decoding after a graph run, graph or not
    Q2, K2, V2 = _inputs(q, k, v, P + T, 4, F, group)
    go2, gsel2 = cs.decode_run(gs, Q2, K2, V2)
    for t in range(4):
        bo, bsel = cs.decode_batch(bs, Q2[t], K2[t], V2[t])
        kk = cs.keep_count(rho, P + T + t)
        assert np.array_equal(gsel2[t, :, :kk], bsel[:, :kk]) and np.array_equal(go2[t], bo), t


def test_graph_run_matches_reference(ctx, ref_ok):
    """One GQA-4 session: every step's set equals the reference's decode_step
    (period 8 reuse of the cached accumulator), outputs within 1e-3."""
    P, d, T, g = 4096, 128, 10, 4
    rc = cs.RetrievalConfig(keep_ratio=0.2, search_period=8)
    q, k, v = workload(P, T, d, seed=72)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=32, seed=1, score_bits=32)
    qq = np.concatenate([q[:P]] * g)
    s = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=g, max_decode_steps=T)
    r = ob.RefSession.prefill(qq, k[:P], v[:P], widths, ic, rc, g)
    Q = np.stack([np.stack([q[P + t]] * g) for t in range(T)])
    out, sel = cs.decode_run([s], Q, k[P:P + T][:, None], v[P:P + T][:, None])
    worst = 0.0
    for t in range(T):
        for h, (rs, ro, _, _) in enumerate(r.step(Q[t], k[P + t], v[P + t])):
            assert np.array_equal(sel[t, h, :len(rs)], rs), (t, h)
            worst = max(worst, rel_err(out[t, h], ro))
    assert worst <= 1e-3, worst
    assert tables_equal(s.export_index(), r.export())


def test_graph_run_k_override_and_device_tensors(ctx):
    torch = pytest.importorskip("torch")
    P, d, T, F = 4096, 64, 6, 2
    rc = cs.RetrievalConfig()
    q, k, v, base, gs, bs = _setup(ctx, P, d, T, 1, rc, F, seed=73)
    Q, K, V = _inputs(q, k, v, P, T, F, 1)
    ko = np.array([[50 + 7 * t + f for f in range(F)] for t in range(T)], np.uint64)
    dev = torch.device("cuda:0")
    go, gsel = cs.decode_run(gs, torch.from_numpy(Q).to(dev), torch.from_numpy(K).to(dev),
                             torch.from_numpy(V).to(dev), k_override=ko)
    go, gsel = go.cpu().numpy(), gsel.cpu().numpy().view(np.uint32)
    hs = [s for s in bs]
    for t in range(T):
        for f, s in enumerate(hs):
            rep = s.decode_step(Q[t][f:f + 1], K[t][f], V[t][f], k_override=int(ko[t, f]))
            rep = rep[0] if isinstance(rep, list) else rep
            assert rep.k == int(ko[t, f])
            assert np.array_equal(gsel[t, f, :rep.k], rep.selected), (t, f)
            assert np.array_equal(go[t, f], rep.output), (t, f)


def test_graph_run_refuses_without_state_change(ctx):
    P, d, T = 2048, 64, 4
    q, k, v = workload(P, T + 2, d, seed=74)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=32)
    s = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, cs.RetrievalConfig(), max_decode_steps=T)
    img = s.serialize()
    Q = np.stack([q[P + t][None] for t in range(T + 1)])
    with pytest.raises(cs.CapacityError):
        cs.decode_run([s], Q, k[P:P + T + 1][:, None], v[P:P + T + 1][:, None])
    assert s.context_len == P and s.serialize() == img
    bad = k[P:P + T][:, None].copy()
    bad[2, 0, 5] = np.nan
    with pytest.raises(cs.DataError):
        cs.decode_run([s], Q[:T], bad, v[P:P + T][:, None])
    assert s.context_len == P and s.serialize() == img
    out, sel = cs.decode_run([s], Q[:T], k[P:P + T][:, None], v[P:P + T][:, None])
    assert s.context_len == P + T and np.isfinite(out).all()
