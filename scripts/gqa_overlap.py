# diagnostics: overlap of the 4 query heads' selected sets per session (c3 data)
import numpy as np

import bench
import paper_2604_08584_b200 as cs

P = 131072
ctx = cs.Context(0)
widths = [bench.D // bench.M] * bench.M
for g in (0, 3):
    q, k, v = bench.gen_head(cs, g, P + 8)
    pooled = np.ascontiguousarray(np.concatenate([q[:P, r] for r in range(bench.GROUP)]))
    ic = cs.IndexConfig(alpha=0.2, centroids=bench.C_CENT, seed=bench.mix_seed(1, g), score_bits=32)
    s = cs.prefill(ctx, pooled, k[:P], v[:P], widths, ic, cs.RetrievalConfig(), group=4, max_decode_steps=8)
    for t in range(3):
        reps = s.decode_step(q[P + t], k[P + t], v[P + t])
        sets = [set(r.selected.tolist()) for r in reps]
        u = set().union(*sets)
        print(f"head {g} step {t}: K={len(sets[0])} union={len(u)} sum={sum(map(len, sets))} "
              f"load ratio={len(u) / sum(map(len, sets)):.3f}")
