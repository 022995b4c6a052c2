"""Mixed-mode select (tail split): when a batch's problems do not fill whole
rounds of the select grid, the problems past the last full round are cut
into tile pieces spread over all CTAs (a batch smaller than the grid: every
problem); the CTA finishing a problem's last piece merges the pieces'
histograms and logs and finalises it inside the select kernel. CSATTN_SELECT_SMS shrinks the grid so small batches take that
path. Every selected set must equal the reference's (oracle/_ref) decode of
the same fork, outputs within 1e-3, tables equal after the inserts; also with
the speculative cut forced to fail (retry pass over split problems) and with
CSATTN_TAIL_SPLIT=0 (plain rounds)."""
import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from oracle import bindings as ob
from tests.helpers import rel_err, tables_equal, workload

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_ref():
    if not ob.ref_available():
        pytest.skip("oracle/_ref not built")


@pytest.mark.parametrize("P,F,sms,env", [
    (20000, 11, 8, {}),                            # 44 problems, grid 16: 2 rounds + 12 split problems (5 tiles each)
    (9000, 9, 4, {}),                              # 36 problems, grid 8: 4 rounds + 4 split problems
    (20000, 11, 8, {"CSATTN_SPEC_KEEP": "2.0"}),   # every speculative cut fails: retry pass
    (20000, 11, 8, {"CSATTN_TAIL_SPLIT": "0"}),    # tail split off: plain rounds
    (20000, 11, 8, {"CSATTN_ATT_GQA": "1"}),       # + the opt-in warp-per-head (GQA) attention
    (20000, 11, 64, {}),                           # small batch (44 < 128 slots): every problem in pieces
    (20000, 11, 64, {"CSATTN_SMALL_MIXED": "0"}),  # small batch: part units + select_merge_kernel
    (20000, 11, 64, {"CSATTN_SPEC_KEEP": "2.0"}),  # small batch, all pieces' speculation fails
    (20000, 11, 8, {"rc": "period4"}),             # cached candidate scores on non-search steps
    (20000, 11, 64, {"rc": "period4"}),
    (20000, 11, 8, {"rc": "no_passthrough"}),      # window keys compete at score 0
    (20000, 11, 64, {"rc": "no_passthrough"}),
    # route -> select programmatic launch (default here: select starts at route's start)
    (20000, 11, 8, {"CSATTN_PDL": "0"}),                             # off
    (20000, 11, 8, {"CSATTN_PDL": "2", "CSATTN_SPEC_KEEP": "2.0"}),  # trigger once lists are known, + retry pass
    (20000, 11, 64, {"CSATTN_PDL": "3", "CSATTN_SPEC_KEEP": "2.0"}), # trigger at route's exit, + retry pass
])
def test_tail_split_batch_equals_reference(monkeypatch, P, F, sms, env):
    monkeypatch.setenv("CSATTN_SELECT_SMS", str(sms))
    monkeypatch.setenv("CSATTN_FUSED", "0")
    for key, val in env.items():
        if key != "rc":
            monkeypatch.setenv(key, val)
    gqa = "CSATTN_ATT_GQA" in env
    rc_kw = {"period4": dict(search_period=4, keep_ratio=0.15),
             "no_passthrough": dict(recent_passthrough=False)}.get(env.get("rc"), {})
    ctx = cs.Context(0)
    T, d = 4, (128 if gqa else 64)  # the warp-per-head attention is the d = 128 kernel
    q, k, v = workload(P, 32, d, seed=P + F)
    widths = cs.uniform_widths(d, 4)
    ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=32)
    rc = cs.RetrievalConfig(**{"keep_ratio": 0.05, **rc_kw})
    qq = np.ascontiguousarray(np.concatenate([q[:P]] * 4))
    base = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=4, max_decode_steps=T)
    batch = [base.fork(T) for _ in range(F)]
    rbase = ob.RefSession.prefill(qq, k[:P], v[:P], widths, ic, rc, 4)
    assert tables_equal(base.export_index(), rbase.export())
    rsess = [rbase.fork() for _ in range(F)]
    rng = np.random.default_rng(3)
    worst = 0.0
    for t in range(T):
        Q = np.stack([q[(P + 5 * f + t + 7 * h) % (P + 32)] for f in range(F) for h in range(4)]).astype(np.float32)
        Q *= (1.0 + 0.1 * rng.standard_normal((len(Q), 1))).astype(np.float32)
        Kn = np.stack([k[P + (f + t) % 32] for f in range(F)])
        Vn = np.stack([v[P + (f + 2 * t) % 32] for f in range(F)])
        out, sel = cs.decode_batch(batch, Q, Kn, Vn)
        for f in range(F):
            res = rsess[f].step(Q[4 * f:4 * f + 4], Kn[f], Vn[f])
            for h, (rsel, rout, _, _) in enumerate(res):
                row = 4 * f + h
                assert np.array_equal(sel[row, :len(rsel)], rsel), (t, f, h)
                worst = max(worst, rel_err(out[row], rout))
    assert worst <= 1e-3, worst
    for f in (0, F - 1):
        assert tables_equal(batch[f].export_index(), rsess[f].export())
