"""Table build at the c3 session shape (P = 131072, d = 128, m = 8, C = 64,
alpha = 0.2) from fixed centroids: tcgen05 screen vs plain fp64 kernels,
wall time around the synchronous build (diagnostics, not a bench value)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_08584_b200 as cs  # noqa: E402
from tests.helpers import random_centroids  # noqa: E402

P, d, m, C = 131072, 128, 8, 64
rng = np.random.default_rng(0)
k = rng.standard_normal((P, d)).astype(np.float32)
v = rng.standard_normal((P, d)).astype(np.float32)
widths = cs.uniform_widths(d, m)
cent = random_centroids(widths, C, 1)
ic = cs.IndexConfig(alpha=0.2, centroids=C, score_bits=32)
res = {}
for mode in sys.argv[1:] or ["tc", "fp64", "tc"]:
    if mode == "fp64":
        os.environ["CSATTN_BUILD"] = "fp64"
    else:
        os.environ.pop("CSATTN_BUILD", None)
    ctx = cs.Context(0)
    t0 = time.perf_counter()
    g = cs.prefill_from_centroids(ctx, cent, k, v, widths, ic, cs.RetrievalConfig())
    t1 = time.perf_counter()
    print(f"{mode}: build {1e3 * (t1 - t0):.2f} ms (incl. 128 MB KV upload), stats {ctx.build_stats}", flush=True)
    res[mode] = g.export_index()
if "tc" in res and "fp64" in res:
    same = all(np.array_equal(a, b) for a, b in zip(res["tc"], res["fp64"]))
    print("tables identical:", same)
