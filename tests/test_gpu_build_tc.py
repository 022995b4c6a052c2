"""The tcgen05 table build (build_tc.cu): a tf32 tensor-core screen of every
(key, table) pair plus an exact fp64 rescore of the candidates. Its tables
must be bit-identical to the reference's (oracle/_ref) and to the plain fp64
build (CSATTN_BUILD=fp64); the context's build stats prove the tensor-core
path ran (not the fallback), and a forced-inconclusive screen
(CSATTN_BUILD_QMARGIN < 0: theta above the true L-th score) must fall back
to the fp64 kernels with the same tables."""
import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from oracle import bindings as ob
from tests.helpers import random_centroids, tables_equal, workload

pytestmark = pytest.mark.gpu


def _ref():
    return ob.RefSession if ob.ref_available() else ob.OraSession


def _build(monkeypatch, mode, cent, k, v, widths, ic, margin=None):
    if mode:
        monkeypatch.setenv("CSATTN_BUILD", mode)
    else:
        monkeypatch.delenv("CSATTN_BUILD", raising=False)
    if margin is None:
        monkeypatch.delenv("CSATTN_BUILD_QMARGIN", raising=False)
    else:
        monkeypatch.setenv("CSATTN_BUILD_QMARGIN", str(margin))
    ctx = cs.Context(0)
    g = cs.prefill_from_centroids(ctx, cent, k, v, widths, ic, cs.RetrievalConfig())
    return ctx, g


CASES = [
    # P, d, m, C, alpha, normalize
    (4096, 64, 4, 16, 0.2, False),
    (5000, 64, 8, 32, 0.1, True),       # ragged last tile, 8-wide subspaces
    (20000, 128, 8, 64, 0.2, False),    # c3-shaped subspaces
    (20000, 128, 8, 64, 0.2, True),
    (12345, 128, 4, 128, 0.05, False),  # 32-wide subspaces, C = 128 (one per TMEM pass... two)
    (3000, 96, 6, 48, 0.5, False),      # d not a multiple of 32, C = 48
]


@pytest.mark.parametrize("P,d,m,C,alpha,normalize", CASES)
def test_tc_build_equals_reference(monkeypatch, P, d, m, C, alpha, normalize):
    q, k, v = workload(P, 1, d, seed=P + d)
    k, v = np.ascontiguousarray(k[:P]), np.ascontiguousarray(v[:P])
    widths = cs.uniform_widths(d, m)
    cent = random_centroids(widths, C, 5)
    ic = cs.IndexConfig(alpha=alpha, centroids=C, score_bits=32, normalize_keys=normalize)
    ctx, g = _build(monkeypatch, None, cent, k, v, widths, ic)
    tc, fb = ctx.build_stats
    assert tc == 1 and fb == 0, (tc, fb)
    r = _ref().from_centroids(cent, k, v, widths, ic, cs.RetrievalConfig())
    assert tables_equal(g.export_index(), r.export())
    ctx2, g2 = _build(monkeypatch, "fp64", cent, k, v, widths, ic)
    assert ctx2.build_stats == (0, 0)
    a, b = g.export_index(), g2.export_index()
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_tc_build_heavy_ties_and_zero_keys(monkeypatch):
    """Duplicate and zero key slices: many equal scores at the threshold."""
    P, d, C = 6000, 64, 16
    rng = np.random.default_rng(7)
    base = rng.standard_normal((50, d)).astype(np.float32)
    k = base[rng.integers(0, 50, P)].copy()
    k[::7, :16] = 0.0
    v = rng.standard_normal((P, d)).astype(np.float32)
    widths = cs.uniform_widths(d, 4)
    cent = random_centroids(widths, C, 2)
    for normalize in (False, True):
        ic = cs.IndexConfig(alpha=0.2, centroids=C, score_bits=32, normalize_keys=normalize)
        ctx, g = _build(monkeypatch, None, cent, k, v, widths, ic)
        r = _ref().from_centroids(cent, k, v, widths, ic, cs.RetrievalConfig())
        assert tables_equal(g.export_index(), r.export())
        assert ctx.build_stats[0] == 1


def test_tc_build_inconclusive_screen_falls_back(monkeypatch):
    """theta forced far above the L-th score: the count check fails, the
    session is rebuilt by the fp64 kernels, tables still exact."""
    P, d, C = 8192, 64, 16
    q, k, v = workload(P, 1, d, seed=3)
    k, v = np.ascontiguousarray(k[:P]), np.ascontiguousarray(v[:P])
    widths = cs.uniform_widths(d, 4)
    cent = random_centroids(widths, C, 4)
    ic = cs.IndexConfig(alpha=0.2, centroids=C, score_bits=32)
    ctx, g = _build(monkeypatch, None, cent, k, v, widths, ic, margin=-0.15)
    assert ctx.build_stats == (1, 1)
    r = _ref().from_centroids(cent, k, v, widths, ic, cs.RetrievalConfig())
    assert tables_equal(g.export_index(), r.export())


def test_tc_build_prefill_batch_kmeans(monkeypatch):
    """The full prefill (GPU k-means, GQA pooling) through the tc build."""
    P, d, group = 8192, 128, 2
    q, k, v = workload(P, 1, d)
    qq = np.concatenate([q[:P]] * group)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=32, seed=1, score_bits=32)
    rc = cs.RetrievalConfig()
    monkeypatch.delenv("CSATTN_BUILD", raising=False)
    ctx = cs.Context(0)
    g = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=group)
    assert ctx.build_stats == (1, 0)
    r = _ref().prefill(qq, k[:P], v[:P], widths, ic, rc, group)
    assert tables_equal(g.export_index(), r.export())


def test_tc_build_negative_zero_scores(monkeypatch):
    """Denormal key slices: dots of magnitude < half the smallest subnormal
    round to -0.0f / +0.0f. With alpha = 0.6 the threshold is negative, so the
    zero scores are table members; the tables keep the reference's float(s)
    bits (the -0.0 sign included) while ranking treats -0.0 == +0.0."""
    P, d, C = 6000, 64, 16
    rng = np.random.default_rng(11)
    k = rng.standard_normal((P, d)).astype(np.float32)
    tiny = np.float32(1.4e-45)
    sgn = np.where(rng.random((P // 5, 16)) < 0.5, -1, 1).astype(np.float32)
    k[::5, :16] = tiny * sgn
    v = rng.standard_normal((P, d)).astype(np.float32)
    widths = cs.uniform_widths(d, 4)
    cent = random_centroids(widths, C, 6)
    ic = cs.IndexConfig(alpha=0.6, centroids=C, score_bits=32)
    ctx, g = _build(monkeypatch, None, cent, k, v, widths, ic)
    assert ctx.build_stats == (1, 0)
    a = g.export_index()
    r = _ref().from_centroids(cent, k, v, widths, ic, cs.RetrievalConfig())
    assert tables_equal(a, r.export())
    neg0 = sum(int(np.count_nonzero(a[2][t, :a[0][t]].view(np.uint32) == 0x80000000)) for t in range(len(a[0])))
    assert neg0 > 0, "the case must exercise -0.0 table scores"
