"""Generate tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libcsattn_ref.so, built from /root/reference/proj/src by
oracle/Makefile). TEST INFRASTRUCTURE: run here, where /root/reference exists;
the fixtures travel with the repo so the C restatement and the CUDA path stay
pinned to the reference's own outputs on boxes without it.

usage: python tests/golden/make_golden.py
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2604_08584_b200 as cs  # noqa: E402  (host-side generator only)
from oracle import bindings as ob  # noqa: E402

# (name, P, T, d, m, C, alpha, seed, group, schedule rho/period, window, passthrough)
CASES = [
    ("c1_head", 4096, 6, 128, 8, 64, 0.2, 2026, 1, 0.05, 1, 32, True),   # BASELINE config 1
    ("gqa4_small", 1024, 5, 64, 4, 16, 0.25, 7, 4, 0.05, 1, 16, True),
    ("period4_nopt", 768, 6, 32, 4, 8, 0.5, 11, 1, 0.15, 4, 8, False),
]


def table_digest(lens, idx, sc):
    """sha256 over the tables in TopList order: per table its length, indices
    and score bits (the fixtures stay small; any difference changes it)."""
    h = hashlib.sha256()
    for t in range(len(lens)):
        n = int(lens[t])
        h.update(np.uint32(n).tobytes())
        h.update(np.ascontiguousarray(idx[t, :n], np.uint32).tobytes())
        h.update(np.ascontiguousarray(sc[t, :n], np.float32).view(np.uint32).tobytes())
    return h.digest()


def main():
    if not ob.ref_available():
        raise SystemExit("oracle/_ref/libcsattn_ref.so missing: make -C oracle (needs /root/reference)")
    out = os.path.dirname(os.path.abspath(__file__))
    for (name, P, T, d, m, C, alpha, seed, group, rho, period, window, pt) in CASES:
        q, k, v = cs.make_synthetic(cs.SyntheticSpec(rows=P + T, dim=d, clusters=8, seed=seed))
        if group > 1:  # head h sees the same keys with its own dwell
            qs = [cs.make_synthetic(cs.SyntheticSpec(rows=P + T, dim=d, clusters=8, seed=seed,
                                                     dwell=dw))[0] for dw in (32, 16, 64, 8)[:group]]
            qg = np.stack(qs, 1)  # [rows, group, d]
            pooled = np.ascontiguousarray(np.concatenate([qg[:P, h] for h in range(group)]))
        else:
            qg = q[:, None, :]
            pooled = q[:P]
        widths = cs.uniform_widths(d, m)
        ic = cs.IndexConfig(alpha=alpha, centroids=C, iterations=10, seed=1, score_bits=32)
        rc = cs.RetrievalConfig(keep_ratio=rho, search_period=period, recent_window=window,
                                recent_passthrough=pt)
        ref = ob.RefSession.prefill(pooled, k[:P], v[:P], widths, ic, rc, group)
        lens0, idx0, sc0, cent = ref.export()
        sels, outs, ks = [], [], []
        for t in range(T):
            res = ref.step(qg[P + t], k[P + t], v[P + t])
            for h, (sel, o, _, rep) in enumerate(res):
                sels.append(np.asarray(sel, np.uint32))
                outs.append(o)
                ks.append(len(sel))
        lens1, idx1, sc1, _ = ref.export()
        np.savez_compressed(
            os.path.join(out, f"{name}.npz"),
            P=P, T=T, d=d, m=m, C=C, alpha=alpha, seed=seed, group=group, rho=rho,
            period=period, window=window, passthrough=int(pt), centroids=cent,
            tables0=np.frombuffer(table_digest(lens0, idx0, sc0), np.uint8),
            tables1=np.frombuffer(table_digest(lens1, idx1, sc1), np.uint8),
            k=np.asarray(ks, np.int64), selected=np.concatenate(sels), outputs=np.stack(outs))
        print(f"{name}: tables {len(lens0)}, steps {T} x {group} heads, "
              f"sum K {sum(ks)} -> {name}.npz")


if __name__ == "__main__":
    main()
