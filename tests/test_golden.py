"""Golden fixtures from the reference library itself (tests/golden/make_golden.py):
the C restatement (CPU) and the CUDA path (GPU) must reproduce the reference's
tables (digest), selected sets (exact) and outputs (<= 1e-3 rel) without
/root/reference being present."""
import glob
import os
import sys

import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from oracle import bindings as ob
from tests.helpers import rel_err

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_golden import table_digest  # noqa: E402

CASES = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))


def _inputs(g):
    P, T, d, seed, group = int(g["P"]), int(g["T"]), int(g["d"]), int(g["seed"]), int(g["group"])
    q, k, v = cs.make_synthetic(cs.SyntheticSpec(rows=P + T, dim=d, clusters=8, seed=seed))
    if group > 1:
        qs = [cs.make_synthetic(cs.SyntheticSpec(rows=P + T, dim=d, clusters=8, seed=seed,
                                                 dwell=dw))[0] for dw in (32, 16, 64, 8)[:group]]
        qg = np.stack(qs, 1)
        pooled = np.ascontiguousarray(np.concatenate([qg[:P, h] for h in range(group)]))
    else:
        qg, pooled = q[:, None, :], q[:P]
    widths = cs.uniform_widths(d, int(g["m"]))
    ic = cs.IndexConfig(alpha=float(g["alpha"]), centroids=int(g["C"]), iterations=10, seed=1,
                        score_bits=32)
    rc = cs.RetrievalConfig(keep_ratio=float(g["rho"]), search_period=int(g["period"]),
                            recent_window=int(g["window"]),
                            recent_passthrough=bool(int(g["passthrough"])))
    return P, T, group, qg, pooled, k, v, widths, ic, rc


def _check_run(g, export0, steps, export1):
    assert table_digest(*export0[:3]) == g["tables0"].tobytes(), "prefill tables differ"
    off = 0
    for i, (sel, out) in enumerate(steps):
        kk = int(g["k"][i])
        assert len(sel) == kk, (i, len(sel), kk)
        assert np.array_equal(np.asarray(sel, np.uint32), g["selected"][off:off + kk]), i
        assert rel_err(out, g["outputs"][i]) <= 1e-3, i
        off += kk
    assert table_digest(*export1[:3]) == g["tables1"].tobytes(), "tables differ after inserts"


@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(c)[:-4] for c in CASES])
def test_restatement_reproduces_reference_golden(path):
    g = np.load(path)
    P, T, group, qg, pooled, k, v, widths, ic, rc = _inputs(g)
    o = ob.OraSession.prefill(pooled, k[:P], v[:P], widths, ic, rc, group)
    e0 = o.export()
    steps = []
    for t in range(T):
        for sel, out, _, _ in o.step(qg[P + t], k[P + t], v[P + t]):
            steps.append((sel, out))
    _check_run(g, e0, steps, o.export())


@pytest.mark.gpu
@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(c)[:-4] for c in CASES])
def test_cuda_path_reproduces_reference_golden(ctx, path):
    g = np.load(path)
    P, T, group, qg, pooled, k, v, widths, ic, rc = _inputs(g)
    s = cs.prefill(ctx, pooled, k[:P], v[:P], widths, ic, rc, group=group, max_decode_steps=T)
    e0 = s.export_index()
    steps = []
    for t in range(T):
        res = s.decode_step(qg[P + t], k[P + t], v[P + t])
        res = res if isinstance(res, list) else [res]
        steps.extend((r.selected, r.output) for r in res)
    _check_run(g, e0, steps, s.export_index())
