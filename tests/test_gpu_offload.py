"""The CPU<->GPU offload mode: with the context's KV
placement set to pinned host memory, every KV row (prefill and appended) lives
in mapped host memory and the kernels read only the selected rows across the
host link. Results must not change: the same parity bar as the HBM path."""
import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from oracle import bindings as ob
from tests.helpers import lockstep, tables_equal, workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def host_ctx():
    c = cs.Context(0)
    c.set_kv_placement("host")
    yield c
    c.close()


@pytest.mark.parametrize("group", [1, 4])
def test_offload_decode_matches_reference(host_ctx, group):
    P, T, d = 4096, 24, 128
    q, k, v = workload(P, T, d, seed=61)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=32, seed=1, score_bits=32)
    rc = cs.RetrievalConfig()
    qq = np.concatenate([q[:P]] * group) if group > 1 else q[:P]
    g = cs.prefill(host_ctx, qq, k[:P], v[:P], widths, ic, rc, group=group, max_decode_steps=T)
    r = ob.RefSession.prefill(qq, k[:P], v[:P], widths, ic, rc, group)
    assert tables_equal(g.export_index(), r.export())
    lockstep(g, r, q, k, v, P, T, group=group, check_tables_every=8)


def test_offload_forks_batch_and_image(host_ctx, ctx):
    """Forks share the host-resident prefill rows; a batch step over forks and
    the CSAT image equal those of the HBM-resident session."""
    P, T, d = 2048, 6, 64
    q, k, v = workload(P, T, d, seed=62)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=32)
    rc = cs.RetrievalConfig()
    h = cs.prefill(host_ctx, q[:P], k[:P], v[:P], widths, ic, rc, max_decode_steps=T)
    dv = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, rc, max_decode_steps=T)
    hf = [h.fork() for _ in range(3)]
    df = [dv.fork() for _ in range(3)]
    for t in range(T):
        Q = np.stack([q[P + t] * (1 + 0.1 * i) for i in range(3)]).astype(np.float32)
        K = np.stack([k[P + t]] * 3)
        V = np.stack([v[P + t]] * 3)
        ho, hs = cs.decode_batch(hf, Q, K, V)
        do, ds = cs.decode_batch(df, Q, K, V)
        kk = cs.keep_count(0.05, P + t)  # row r's set is sel[r, :K]
        assert np.array_equal(hs[:, :kk], ds[:, :kk])
        assert np.array_equal(ho, do)
    assert hf[0].serialize() == df[0].serialize()
    kh, vh = hf[1].read_kv(0, P + T)
    kd, vd = df[1].read_kv(0, P + T)
    assert np.array_equal(kh, kd) and np.array_equal(vh, vd)
