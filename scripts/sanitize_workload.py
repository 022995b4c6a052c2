"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every decode kernel on both select paths plus the table build.
  * prefill of a GQA-4 session at P = 4096 (k-means full batch, build_scores,
    build_lists),
  * 2 decode steps of 80 forks in one batch (320 problems: the persistent
    non-split select with speculation, the retry pass, 512-row attend chunks),
  * 2 decode steps of 2 forks (8 problems: the fused cluster step, with the
    insert as its programmatic dependent; CSATTN_FUSED=0 takes the mixed
    select pieces instead),
  * a search_period = 4 session (candidate cache store / reuse).
Run: compute-sanitizer --tool <t> python scripts/sanitize_workload.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_08584_b200 as cs  # noqa: E402

P, d, G = 4096, 128, 4
ctx = cs.Context(0)
q, k, v = cs.make_synthetic(cs.SyntheticSpec(rows=P + 400, dim=d, clusters=8, seed=5))
widths = cs.uniform_widths(d, 8)
ic = cs.IndexConfig(alpha=0.2, centroids=32, seed=1, score_bits=32)
rc = cs.RetrievalConfig()
qq = np.ascontiguousarray(np.concatenate([q[:P]] * G))
base = cs.prefill(ctx, qq, k[:P], v[:P], widths, ic, rc, group=G, max_decode_steps=4)
for nf in (80, 2):
    forks = [base.fork(4) for _ in range(nf)]
    for t in range(2):
        Q = np.stack([q[P + f + t] for f in range(nf) for _ in range(G)])
        out, sel = cs.decode_batch(forks, Q, k[P + t:P + t + nf], v[P + t:P + t + nf])
        assert np.isfinite(out).all()
    del forks
s4 = cs.prefill(ctx, q[:P], k[:P], v[:P], widths, ic, cs.RetrievalConfig(search_period=4),
                max_decode_steps=6)
for t in range(6):
    s4.decode_step(q[P + t], k[P + t], v[P + t])
ctx.synchronize()
print("sanitize workload done, launches", ctx.launches)
