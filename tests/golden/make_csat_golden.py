"""Generate tests/golden/csat_*.bin: CSAT v1 index images written by the
UNMODIFIED reference's serialize_index (index.cpp:289-318), built with
build_index over the reference generator's synthetic rows
(oracle/_ref/libcsattn_ref.so). TEST INFRASTRUCTURE: run here, where
/root/reference exists; the images travel with the repo so the codec
(csat.cpp) and the device writer (csat_dev.cu) stay pinned without it.

usage: python tests/golden/make_csat_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2604_08584_b200 as cs  # noqa: E402  (host-side generator only)
from oracle import bindings as ob  # noqa: E402

# (name, P, d, m, C, alpha, synthetic seed, normalize_keys)
CASES = [("csat_small", 1024, 64, 4, 16, 0.25, 91, False),
         ("csat_norm", 512, 32, 4, 8, 0.5, 92, True)]


def build(P, d, m, C, alpha, seed, normalize):
    q, k, v = cs.make_synthetic(cs.SyntheticSpec(rows=P, dim=d, clusters=8, seed=seed))
    ic = cs.IndexConfig(alpha=alpha, centroids=C, seed=1, score_bits=32, normalize_keys=normalize)
    return ob.RefSession.prefill(q, k, v, cs.uniform_widths(d, m), ic, cs.RetrievalConfig())


def serialize(ref, bits):
    import ctypes as C
    L = ob.ref_lib()
    n = C.c_uint64()
    assert L.csref_serialize(ref.h, bits, None, 0, C.byref(n)) == 0
    buf = (C.c_uint8 * n.value)()
    assert L.csref_serialize(ref.h, bits, buf, n.value, C.byref(n)) == 0
    return bytes(buf)


def main():
    out = os.path.dirname(os.path.abspath(__file__))
    for name, P, d, m, C, alpha, seed, norm in CASES:
        ref = build(P, d, m, C, alpha, seed, norm)
        for bits in (32, 16):
            with open(os.path.join(out, f"{name}_{bits}.bin"), "wb") as f:
                f.write(serialize(ref, bits))
        print(name, "written")


if __name__ == "__main__":
    main()
