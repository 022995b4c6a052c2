"""Shared workload builders for the parity tests (seeded, reference generator)."""
from __future__ import annotations

import numpy as np

import paper_2604_08584_b200 as cs
from oracle import bindings as ob


def workload(P: int, T: int, d: int, seed: int = 2026, dwell: int = 32):
    spec = cs.SyntheticSpec(rows=P + T, dim=d, clusters=8, seed=seed, dwell=dwell)
    return cs.make_synthetic(spec)


def random_centroids(widths, c, seed):
    """Unit centroid rows packed per subspace (test_retrieval.cpp:30-45 style)."""
    rng = np.random.default_rng(seed)
    out = []
    for w in widths:
        x = rng.standard_normal((c, w)).astype(np.float32)
        for j in range(c):
            ob.ora_lib().ora_l2_normalize(x[j].ctypes.data, w)
        out.append(x.reshape(-1))
    return np.concatenate(out)


def tables_equal(a, b):
    la, ia, sa, ca = a
    lb, ib, sb, cb = b
    if not np.array_equal(la, lb) or not np.array_equal(ca, cb):
        return False
    for t in range(len(la)):
        n = la[t]
        if not (np.array_equal(ia[t, :n], ib[t, :n]) and
                np.array_equal(sa[t, :n].view(np.uint32), sb[t, :n].view(np.uint32))):
            return False
    return True


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def lockstep(gpu: cs.Session, ref, q, k, v, P, T, group=1, check_tables_every=0, tol=1e-3,
             want_weights=True):
    """Drive the GPU session and a CPU checker through T identical steps.
    With the reference library as checker, the accumulated candidate sets
    (reduce_by_key output, SearchState::cached) are compared bit-exactly too."""
    d = k.shape[1]
    worst = 0.0
    check_cand = hasattr(ref, "candidates")
    if check_cand:
        gpu.keep_candidates(True)
    for t in range(T):
        qs = np.stack([q[P + t]] * group) if q.ndim == 2 else q[t]
        g = gpu.decode_step(qs, k[P + t], v[P + t], want_weights=want_weights)
        g = g if isinstance(g, list) else [g]
        r = ref.step(qs, k[P + t], v[P + t])
        if check_cand:
            for h in range(group):
                gi, gs = gpu.candidates(h)
                ri, rs = ref.candidates(h)
                assert np.array_equal(gi, ri), (t, h, "candidate keys",
                                                np.setxor1d(gi, ri)[:8])
                bad = np.nonzero(gs.view(np.uint64) != rs.view(np.uint64))[0]
                assert bad.size == 0, (t, h, "candidate scores", gi[bad[:4]], gs[bad[:4]],
                                       rs[bad[:4]])
        for h, (gr, (sel, out, wts, rep)) in enumerate(zip(g, r)):
            assert gr.k == len(sel), (t, h, gr.k, len(sel))
            assert np.array_equal(gr.selected, sel), (t, h, np.setdiff1d(gr.selected, sel)[:8],
                                                      np.setdiff1d(sel, gr.selected)[:8])
            e = rel_err(gr.output, out)
            worst = max(worst, e)
            assert e <= tol, (t, h, e)
            if want_weights:
                assert np.allclose(gr.weights, wts, rtol=1e-3, atol=1e-6), (t, h)
            assert gr.searched == bool(rep.searched)
            assert gr.counters.gathered_entries == rep.gathered_entries, (t, h)
            assert gr.counters.centroid_dot_ops == rep.centroid_dot_ops, (t, h)
            assert gr.counters.inserts_applied == rep.inserts_applied, (t, h)
            assert gr.counters.inserts_attempted == rep.inserts_attempted
            assert gr.counters.attention_key_ops == rep.attention_key_ops
            assert abs(gr.counters.h2d_bytes_model - rep.h2d_bytes_model) <= 1e-9 * max(1.0, rep.h2d_bytes_model)
        if check_tables_every and (t + 1) % check_tables_every == 0:
            assert tables_equal(gpu.export_index(), ref.export()), f"tables diverged at step {t}"
    return worst
