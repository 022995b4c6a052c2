"""k-means + table build of one c3-shaped KV head (P = 131072, GQA 4 -> 524288
pooled query rows, d = 128, m = 8, C = 64): wall time of the synchronous
prefill (diagnostics; CSATTN_KM_PROF=1 adds the seeding phase split)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_08584_b200 as cs  # noqa: E402

P, d, G = 131072, 128, 4
rng = np.random.default_rng(0)
q = rng.standard_normal((G * P, d)).astype(np.float32)
k = rng.standard_normal((P, d)).astype(np.float32)
v = rng.standard_normal((P, d)).astype(np.float32)
ic = cs.IndexConfig(alpha=0.2, centroids=64, seed=1, score_bits=32)
ctx = cs.Context(0)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    t0 = time.perf_counter()
    s = cs.prefill(ctx, q, k, v, cs.uniform_widths(d, 8), ic, cs.RetrievalConfig(), group=G)
    print(f"prefill {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    cent = s.export_index()[3]
    print("centroid checksum", float(np.float64(cent).sum()), flush=True)
