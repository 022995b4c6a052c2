import numpy as np
import paper_2604_08584_b200 as cs
from tests.helpers import workload
hc = cs.Context(0); hc.set_kv_placement("host")
dc = cs.Context(0)
P, T, d = 2048, 6, 64
q, k, v = workload(P, T, d, seed=62)
widths = cs.uniform_widths(d, 8)
ic = cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=32)
rc = cs.RetrievalConfig()
h = cs.prefill(hc, q[:P], k[:P], v[:P], widths, ic, rc, max_decode_steps=T)
dv = cs.prefill(dc, q[:P], k[:P], v[:P], widths, ic, rc, max_decode_steps=T)
print("tables equal", all(np.array_equal(a, b) for a, b in zip(h.export_index()[:3], dv.export_index()[:3])))
hf = [h.fork() for _ in range(3)]; df = [dv.fork() for _ in range(3)]
for t in range(T):
    Q = np.stack([q[P + t] * (1 + 0.1 * i) for i in range(3)]).astype(np.float32)
    K = np.stack([k[P + t]] * 3); V = np.stack([v[P + t]] * 3)
    ho, hs = cs.decode_batch(hf, Q, K, V)
    do, ds = cs.decode_batch(df, Q, K, V)
    kk = cs.keep_count(0.05, P + t)
    print(t, "sel equal", np.array_equal(hs[:, :kk], ds[:, :kk]), "full", np.array_equal(hs, ds), "out", np.abs(ho - do).max())
    if not np.array_equal(hs, ds):
        r = np.nonzero((hs != ds).any(1))[0][0]; c = np.nonzero(hs[r] != ds[r])[0]
        print("  row", r, "cols", c[:5], hs[r, c[:5]], ds[r, c[:5]], "K", kk)
