# diagnostics: first table divergence after loading a 16-bit image (GPU vs reference)
import numpy as np
import paper_2604_08584_b200 as cs
from oracle import bindings as ob
from tests.helpers import workload

ctx = cs.Context(0)
P, T, d = 2048, 24, 64
q, k, v = workload(P, T, d, seed=6)
widths = cs.uniform_widths(d, 8)
ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=16)
rc = cs.RetrievalConfig()
img = ob.RefSession.prefill(q[:P], k[:P], v[:P], widths, ic, rc).serialize(16)
g = cs.deserialize(ctx, img, k[:P], v[:P], rc, max_decode_steps=T)
r = ob.RefSession.load(img, k[:P], v[:P], d, rc)

def tabs(x):
    lens, idx, sc = x[0], x[1], x[2]
    return [(sorted(zip(idx[t, :lens[t]].tolist(), sc[t, :lens[t]].tolist()))) for t in range(len(lens))]

for t in range(T):
    a, b = tabs(g.export_index()), tabs(r.export())
    bad = [i for i in range(len(a)) if a[i] != b[i]]
    if bad:
        i = bad[0]
        sa, sb = set(a[i]), set(b[i])
        print("step", t, "tables differ:", len(bad), "first", i, "gpu-only", sorted(sa - sb)[:5], "ref-only", sorted(sb - sa)[:5])
        lr = r.export()
        n = lr[0][i]
        print("ref tail order", list(zip(lr[1][i, n-6:n].tolist(), lr[2][i, n-6:n].tolist())))
        break
    gg = g.decode_step(q[P + t], k[P + t], v[P + t])
    rr = r.step(q[P + t], k[P + t], v[P + t])
else:
    print("no divergence")
