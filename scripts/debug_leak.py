# diagnostics: context-state leak hunt — a GQA-4 run before a fork batch on the same context
import numpy as np

import paper_2604_08584_b200 as cs
from tests.helpers import workload


def fork_batch(c):
    P, T, d = 2048, 6, 64
    q, k, v = workload(P, T, d, seed=62)
    widths = cs.uniform_widths(d, 8)
    ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=32)
    s = cs.prefill(c, q[:P], k[:P], v[:P], widths, ic, cs.RetrievalConfig(), max_decode_steps=T)
    fs = [s.fork() for _ in range(3)]
    outs = []
    for t in range(T):
        Q = np.stack([q[P + t] * (1 + 0.1 * i) for i in range(3)]).astype(np.float32)
        K = np.stack([k[P + t]] * 3)
        V = np.stack([v[P + t]] * 3)
        outs.append(cs.decode_batch(fs, Q, K, V))
    return outs


def gqa4(c):
    P, T, d = 4096, 24, 128
    q, k, v = workload(P, T, d, seed=61)
    qq = np.concatenate([q[:P]] * 4)
    g = cs.prefill(c, qq, k[:P], v[:P], cs.uniform_widths(d, 8),
                   cs.IndexConfig(alpha=0.2, centroids=32, seed=1, score_bits=32),
                   cs.RetrievalConfig(), group=4, max_decode_steps=T)
    for t in range(T):
        g.decode_step(np.stack([q[P + t]] * 4), k[P + t], v[P + t])
    g.close()


for placement in ("host", "device"):
    ref = fork_batch(cs.Context(0))
    c = cs.Context(0)
    c.set_kv_placement(placement)
    gqa4(c)
    got = fork_batch(c)
    bad = [t for t in range(len(ref)) if not np.array_equal(ref[t][1], got[t][1])]
    print(placement, "steps with different selections:", bad)
    if bad:
        t = bad[0]
        r = np.nonzero((ref[t][1] != got[t][1]).any(1))[0][0]
        cc = np.nonzero(ref[t][1][r] != got[t][1][r])[0]
        print("  step", t, "row", r, "first cols", cc[:6], ref[t][1][r, cc[:6]], got[t][1][r, cc[:6]])
