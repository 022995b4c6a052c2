import numpy as np
import paper_2604_08584_b200 as cs
from tests.helpers import workload
ctx = cs.Context(0)
P, d = 2000, 64
q, k, v = workload(P, 1, d, seed=41)
g = cs.prefill(ctx, q[:P], k[:P], v[:P], cs.uniform_widths(d, 8), cs.IndexConfig(alpha=0.2, centroids=16, seed=1, score_bits=32), cs.RetrievalConfig())
print(g.dense_topk(q[0], 5))
