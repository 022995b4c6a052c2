"""Reference parity at the BENCHMARKED scale (BASELINE configs c2, c3, c5).

The decode step the bench times at 128K (config c3: 131072-key prefill, GQA
groups of 4 pooled into one index per KV head, batch decode of sequences that
fork one prefill) runs machinery that only switches on at scale: the
non-split persistent select (>= 296 problems per launch), the speculative
cut and its retry pass, the 2048-bin histogram over route.cu's score bounds,
512-row attention chunks with 8-row groups, candidate logs sized for the full
context. These tests run exactly that configuration and compare it with the
UNMODIFIED reference (oracle/_ref) on the bench's own synthetic inputs
(SURVEY.md §8(d) seeds and dwells):
  * tables after the GPU build bit-identical to build_index;
  * every checked (sequence, head) selected set identical, output within 1e-3
    (north_star), counters equal;
  * tables bit-identical after the streaming inserts of every step.
Reference semantics: each sequence is an independent Session copy of the
prefilled one (session.hpp:19-31), decode_step per step (session.cpp:46-99).
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from oracle import bindings as ob
from tests.helpers import rel_err, tables_equal

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

D, M, C_CENT, GROUP = 128, 8, 64, 4
DWELLS = (32, 16, 64, 8)
TOL = 1e-3


def mix_seed(seed: int, salt: int) -> int:
    """splitmix64 sub-seed (util.hpp:61-66), as bench.py."""
    mask = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15 * (salt + 1)) & mask
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
    return z ^ (z >> 31)


def kv_head(g: int, rows: int):
    """KV head g of the layer: 4 query streams (dwells), keys, values."""
    seed = mix_seed(2026, g)
    qs, k, v = [], None, None
    for dw in DWELLS:
        q, kk, vv = cs.make_synthetic(cs.SyntheticSpec(rows=rows, dim=D, clusters=8, seed=seed,
                                                       dwell=dw))
        qs.append(q)
        if k is None:
            k, v = kk, vv
    return np.stack(qs, 1), k, v  # q [rows, 4, d]


def pooled(q, P):
    return np.ascontiguousarray(np.concatenate([q[:P, r] for r in range(GROUP)]))


def index_cfg(g):
    return cs.IndexConfig(alpha=0.2, centroids=C_CENT, seed=mix_seed(1, g), score_bits=32)


def check_step(out, sel, row0, ref_res, tag):
    for h, (rs, ro, _, rep) in enumerate(ref_res):
        got = sel[row0 + h, :len(rs)]
        assert np.array_equal(got, rs), (tag, h, np.setdiff1d(got, rs)[:8], np.setdiff1d(rs, got)[:8])
        e = rel_err(out[row0 + h], ro)
        assert e <= TOL, (tag, h, e)
    return max(rel_err(out[row0 + h], ro) for h, (_, ro, _, _) in enumerate(ref_res))


def test_c3_shape_fork_batch_matches_reference(ctx, ref_ok):
    """Config c3 per KV head at full scale: P = 131072, d = 128, m = 8, C = 64,
    alpha = 0.2 (L = 26215), rho = 0.05 (K = 6554), GQA 4 pooled. 80 sequences
    fork the prefill and decode 8 steps in ONE decode_batch each step (320
    problems: the non-split select, as in the bench's 512); sequences 0, 39
    and 79 are stepped by reference Session copies beside it."""
    P, T, F = 131072, 8, 80
    checked = (0, 39, 79)
    q, k, v = kv_head(0, P + F * T)
    widths = cs.uniform_widths(D, M)
    rc = cs.RetrievalConfig()
    pq = pooled(q, P)
    base = cs.prefill(ctx, pq, k[:P], v[:P], widths, index_cfg(0), rc, group=GROUP,
                      max_decode_steps=T)
    ref = ob.RefSession.prefill(pq, k[:P], v[:P], widths, index_cfg(0), rc, GROUP)
    assert base.info().list_capacity == 26215
    assert tables_equal(base.export_index(), ref.export()), "128K GQA-pooled tables differ"
    del pq
    forks = [base] + [base.fork(T) for _ in range(F - 1)]
    refs = {f: ref.fork() for f in checked}
    worst = 0.0
    with ThreadPoolExecutor(max_workers=len(checked)) as ex:
        for t in range(T):
            rows = [P + f * T + t for f in range(F)]
            Q = np.ascontiguousarray(q[rows].reshape(F * GROUP, D))
            Kn, Vn = np.ascontiguousarray(k[rows]), np.ascontiguousarray(v[rows])
            out, sel = cs.decode_batch(forks, Q, Kn, Vn)
            res = dict(zip(checked, ex.map(
                lambda f: refs[f].step(Q[GROUP * f:GROUP * (f + 1)], Kn[f], Vn[f]), checked)))
            assert all(len(r[0][0]) == cs.keep_count(0.05, P + t) for r in res.values())
            for f in checked:
                worst = max(worst, check_step(out, sel, GROUP * f, res[f], (t, f)))
    for f in checked:
        assert tables_equal(forks[f].export_index(), refs[f].export()), f"fork {f} tables after inserts"
    assert worst <= TOL


def test_c2_layer_decode_batch_matches_reference(ctx, ref_ok):
    """Config c2 exactly as the bench runs it: the 8 KV heads of a layer at
    32K, built in one csattn_prefill_batch, then one decode_batch of 8
    sessions x 4 heads per step (32 problems: split part units + merge,
    128-row attention chunks). Every head's tables, selected sets, outputs
    and post-insert tables against 8 reference Sessions."""
    P, T = 32768, 4
    heads = list(range(8))
    with ThreadPoolExecutor(max_workers=8) as ex:
        data = list(ex.map(lambda g: kv_head(g, P + T), heads))
    widths = cs.uniform_widths(D, M)
    rc = cs.RetrievalConfig()
    rows_b = [(pooled(q, P), k[:P], v[:P]) for (q, k, v) in data]
    gpu = cs.prefill_batch(ctx, rows_b, widths, [index_cfg(g) for g in heads], rc, group=GROUP,
                           max_decode_steps=T)
    with ThreadPoolExecutor(max_workers=8) as ex:
        refs = list(ex.map(lambda g: ob.RefSession.prefill(rows_b[g][0], rows_b[g][1], rows_b[g][2],
                                                           widths, index_cfg(g), rc, GROUP), heads))
    for g in heads:
        assert tables_equal(gpu[g].export_index(), refs[g].export()), f"head {g} tables"
    worst = 0.0
    with ThreadPoolExecutor(max_workers=8) as ex:
        for t in range(T):
            Q = np.ascontiguousarray(np.concatenate([data[g][0][P + t] for g in heads]))
            Kn = np.stack([data[g][1][P + t] for g in heads])
            Vn = np.stack([data[g][2][P + t] for g in heads])
            out, sel = cs.decode_batch(gpu, Q, Kn, Vn)
            res = list(ex.map(lambda g: refs[g].step(Q[GROUP * g:GROUP * (g + 1)], Kn[g], Vn[g]), heads))
            for g in heads:
                worst = max(worst, check_step(out, sel, GROUP * g, res[g], (t, g)))
    for g in heads:
        assert tables_equal(gpu[g].export_index(), refs[g].export()), f"head {g} tables after inserts"
    assert worst <= TOL


def test_c5_shape_two_shards_match_reference(ctx, ref_ok):
    """Sequence sharding (config c5's mechanism) against the REFERENCE, not
    against the unsharded GPU path: a 256K-key KV head (GQA 2 pooled) split
    into 2 key-range shards on 2 contexts, the ShardGroup phases with their
    histogram / bucket / count / LSE / victim collectives, 4 steps. The union
    of the shards' selections equals the reference's selected set, outputs
    within 1e-3, and the union of the shards' tables equals the reference's
    tables after the inserts (global TopList semantics)."""
    import torch
    from paper_2604_08584_b200.sharding import ShardGroup

    P, T, grp = 262144, 4, 2
    q, k, v = kv_head(5, P + T)
    widths = cs.uniform_widths(D, M)
    rc = cs.RetrievalConfig()
    pq = np.ascontiguousarray(np.concatenate([q[:P, r] for r in range(grp)]))
    ic = index_cfg(5)
    stream = torch.cuda.Stream()
    ctxs = [cs.Context(0, stream.cuda_stream) for _ in range(2)]
    full = cs.prefill(ctxs[0], pq, k[:P], v[:P], widths, ic, rc, group=grp, max_decode_steps=T)
    ref = ob.RefSession.prefill(pq, k[:P], v[:P], widths, ic, rc, grp)
    assert tables_equal(full.export_index(), ref.export())
    sg = ShardGroup.local(ctxs, [full], max_decode_steps=T)
    full.close()
    for t in range(T):
        K = cs.keep_count(0.05, P + t)
        qs = np.ascontiguousarray(q[P + t, :grp])
        with torch.cuda.stream(stream):
            out, sels = sg.decode_step(torch.from_numpy(qs).cuda(),
                                       torch.from_numpy(k[P + t][None]).cuda(),
                                       torch.from_numpy(v[P + t][None]).cuda(),
                                       want_selected=True, k_max=K)
            out = out.cpu().numpy()
        res = ref.step(qs, k[P + t], v[P + t])
        for h, (rs, ro, _, _) in enumerate(res):
            assert np.array_equal(sels[h], rs), (t, h, np.setxor1d(sels[h], rs)[:8])
            assert rel_err(out[h], ro) <= TOL, (t, h)
    exports = [row[0].export_index() for row in sg.shards]
    rl, ri, rs_, _ = ref.export()
    for tb in range(len(rl)):
        idx = np.concatenate([e[1][tb, :e[0][tb]] for e in exports])
        sc = np.concatenate([e[2][tb, :e[0][tb]] for e in exports])
        order = np.lexsort((idx, -sc.astype(np.float64)))  # TopList order: score desc, index asc
        n = int(rl[tb])
        assert idx.size == n, tb
        assert np.array_equal(idx[order], ri[tb, :n]), tb
        assert np.array_equal(sc[order].view(np.uint32), rs_[tb, :n].view(np.uint32)), tb
