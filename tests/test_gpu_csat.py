"""CSAT v1 images of GPU sessions: the device-written
image is byte-identical to the reference's serialize_index of the same index
(after the build, and after streaming inserts), at 32 and 16 bits; a session
loaded from an image decodes exactly like the reference's load_index session.
Mirrors test_index.cpp:303-358 and acceptance.cpp:425-468 (save -> load ->
identical decode)."""
import glob
import os

import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from oracle import bindings as ob
from tests.helpers import lockstep, workload

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_inputs(name):
    # tests/golden/make_csat_golden.py CASES
    P, d, m, C_, alpha, seed, norm = {"csat_small": (1024, 64, 4, 16, 0.25, 91, False),
                                      "csat_norm": (512, 32, 4, 8, 0.5, 92, True)}[name]
    q, k, v = cs.make_synthetic(cs.SyntheticSpec(rows=P, dim=d, clusters=8, seed=seed))
    return P, d, m, C_, alpha, norm, q, k, v


@pytest.mark.parametrize("name", ["csat_small", "csat_norm"])
@pytest.mark.parametrize("bits", [32, 16])
def test_device_image_equals_reference_golden(ctx, name, bits):
    P, d, m, C_, alpha, norm, q, k, v = _golden_inputs(name)
    ic = cs.IndexConfig(alpha=alpha, centroids=C_, seed=1, score_bits=bits, normalize_keys=norm)
    g = cs.prefill(ctx, q, k, v, cs.uniform_widths(d, m), ic, cs.RetrievalConfig())
    img = g.serialize()
    with open(os.path.join(GOLDEN, f"{name}_{bits}.bin"), "rb") as f:
        assert img == f.read()


@pytest.mark.parametrize("bits", [32, 16])
def test_image_after_streaming_inserts_equals_reference(ctx, bits):
    P, T, d = 2048, 40, 64
    q, k, v = workload(P, T, d, seed=5)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=bits)
    rc = cs.RetrievalConfig()
    g = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, rc, max_decode_steps=T)
    r = ob.RefSession.prefill(q[:P], k[:P], v[:P], widths, ic, rc)
    assert g.serialize() == r.serialize(bits)
    lockstep(g, r, q, k, v, P, T)
    assert g.serialize() == r.serialize(bits)


def _same_index(img_a, img_b):
    """Header, centroids and every table's (index, score) set identical, both in
    descending score order. A 16-bit image written from f32 tables holds runs of
    equal half scores in f32 order; after load_index the reference keeps the
    file's order inside such runs, the device layout (index-sorted) writes them
    in index order. Membership, scores and eviction order are the same."""
    ha, ca, la, ia, sa = cs.csat_decode(img_a)
    hb, cb, lb, ib, sb = cs.csat_decode(img_b)
    assert ha == hb and np.array_equal(ca.view(np.uint32), cb.view(np.uint32))
    assert np.array_equal(la, lb)
    for t in range(len(la)):
        n = int(la[t])
        assert sorted(zip(ia[t, :n].tolist(), sa[t, :n].tolist())) == \
            sorted(zip(ib[t, :n].tolist(), sb[t, :n].tolist())), t
        assert np.all(sa[t, 1:n] <= sa[t, :n - 1]) and np.all(sb[t, 1:n] <= sb[t, :n - 1])


@pytest.mark.parametrize("bits", [32, 16])
def test_loaded_session_decodes_like_reference_load_index(ctx, bits):
    """save -> load -> decode (acceptance.cpp:425-468): both sides load the same
    bytes; selected sets identical, outputs within 1e-3, tables equal after the
    inserts, and the loaded GPU session re-serializes to the same image (up to
    the order inside equal-score runs of a 16-bit image, see _same_index)."""
    P, T, d = 2048, 24, 64
    q, k, v = workload(P, T, d, seed=6)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=bits)
    rc = cs.RetrievalConfig()
    img = ob.RefSession.prefill(q[:P], k[:P], v[:P], widths, ic, rc).serialize(bits)
    g = cs.deserialize(ctx, img, k[:P], v[:P], rc, max_decode_steps=T)
    _same_index(g.serialize(), img)
    if bits == 32:
        assert g.serialize() == img
    r = ob.RefSession.load(img, k[:P], v[:P], d, rc)
    lockstep(g, r, q, k, v, P, T)
    _same_index(g.serialize(), r.serialize(bits))
    if bits == 32:
        assert g.serialize() == r.serialize(bits)


def test_deserialize_validates_rows_and_bytes(ctx):
    P, d = 512, 32
    q, k, v = workload(P, 1, d, seed=7)
    ic = cs.IndexConfig(alpha=0.5, centroids=8, seed=1, score_bits=32)
    g = cs.prefill(ctx, q[:P], k[:P], v[:P], cs.uniform_widths(d, 4), ic, cs.RetrievalConfig())
    img = g.serialize()
    with pytest.raises(cs.ParameterError, match="prefill rows"):
        cs.deserialize(ctx, img, k[:P - 1], v[:P - 1], cs.RetrievalConfig())
    with pytest.raises(cs.BadMagicError):
        cs.deserialize(ctx, b"XSAT" + img[4:], k[:P], v[:P], cs.RetrievalConfig())
    with pytest.raises(cs.TruncatedError, match="byte"):
        cs.deserialize(ctx, img[:len(img) // 2], k[:P], v[:P], cs.RetrievalConfig())
    with pytest.raises(cs.CorruptError, match="trailing"):
        cs.deserialize(ctx, img + b"\0", k[:P], v[:P], cs.RetrievalConfig())
