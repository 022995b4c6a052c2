"""Sequence sharding on one B200: S shards of
every KV-head session on S contexts, collectives as tensor ops. The union of
the shards' selections must equal the unsharded session's selected sets
exactly, outputs agree within 1e-3, and after the streaming inserts the union
of the shards' tables equals the unsharded tables (global TopList semantics)."""
import numpy as np
import pytest

import paper_2604_08584_b200 as cs
from paper_2604_08584_b200.sharding import ShardGroup, shard_bounds
from tests.helpers import rel_err, workload

pytestmark = pytest.mark.gpu


def _union_tables(exports):
    """Merge the shards' exported lists into global TopList order."""
    T = len(exports[0][0])
    lens, idx, sc = [], [], []
    for t in range(T):
        ent = []
        for (l, ix, s, _) in exports:
            ent += [(float(s[t, r]), int(ix[t, r])) for r in range(l[t])]
        ent.sort(key=lambda e: (-e[0], e[1]))
        lens.append(len(ent))
        idx.append([e[1] for e in ent])
        sc.append([e[0] for e in ent])
    return lens, idx, sc


@pytest.mark.parametrize("P,n_shards,group,pt", [(16384, 2, 1, True), (16384, 4, 4, True),
                                                  (12288, 3, 2, False)])
def test_sharded_decode_equals_unsharded(P, n_shards, group, pt):
    import torch
    T, d = 6, 64
    q, k, v = workload(P, T, d, seed=31 + P)
    widths = cs.uniform_widths(d, 4)
    ic = cs.IndexConfig(alpha=0.25, centroids=16, seed=3, score_bits=32)
    rc = cs.RetrievalConfig(keep_ratio=0.05, recent_window=16, recent_passthrough=pt)
    stream = torch.cuda.Stream()
    ctxs = [cs.Context(0, stream.cuda_stream) for _ in range(n_shards)]
    pooled = np.ascontiguousarray(np.concatenate([q[:P]] * group))
    full = cs.prefill(ctxs[0], pooled, k[:P], v[:P], widths, ic, rc, group=group,
                      max_decode_steps=T)
    control = full.fork(T)
    grp = ShardGroup.local(ctxs, [full], max_decode_steps=T)
    assert [b for b in grp.bounds] == shard_bounds(P, n_shards)
    for t in range(T):
        N = P + t
        K = cs.keep_count(0.05, N)
        qs = np.stack([q[P + t]] * group)
        with torch.cuda.stream(stream):
            qd = torch.from_numpy(qs).cuda()
            kd = torch.from_numpy(k[P + t][None]).cuda()
            vd = torch.from_numpy(v[P + t][None]).cuda()
            out, sels = grp.decode_step(qd, kd, vd, want_selected=True, k_max=K)
            out = out.cpu().numpy()
        ref = control.decode_step(qs, k[P + t], v[P + t])
        ref = ref if isinstance(ref, list) else [ref]
        for h in range(group):
            assert np.array_equal(sels[h], ref[h].selected), (t, h, np.setxor1d(sels[h], ref[h].selected)[:8])
            assert rel_err(out[h], ref[h].output) <= 1e-3, (t, h)
    # tables after T inserts: union of the shards == unsharded
    ul, ui, us = _union_tables([row[0].export_index() for row in grp.shards])
    cl, ci, csc, _ = control.export_index()
    assert ul == [int(x) for x in cl]
    for tb in range(len(cl)):
        n = int(cl[tb])
        assert ui[tb] == [int(x) for x in ci[tb, :n]], tb
        assert np.array_equal(np.float32(us[tb]), csc[tb, :n]), tb


def _dist_worker(rank, world, port, P, T, q_out):
    """One rank of ShardGroup.distributed on cuda:0 (gloo, host-staged)."""
    import os
    import torch
    import torch.distributed as dist
    from paper_2604_08584_b200.sharding import HostStagedDist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, group = 64, 2
        q, k, v = workload(P, T, d, seed=77)
        widths = cs.uniform_widths(d, 4)
        ic = cs.IndexConfig(alpha=0.25, centroids=16, seed=3, score_bits=32)
        rc = cs.RetrievalConfig(keep_ratio=0.05, recent_window=16)
        stream = torch.cuda.Stream()
        ctx = cs.Context(0, stream.cuda_stream)
        pooled = np.ascontiguousarray(np.concatenate([q[:P]] * group))
        full = cs.prefill(ctx, pooled, k[:P], v[:P], widths, ic, rc, group=group, max_decode_steps=T)
        control = full.fork(T) if rank == 0 else None
        grp = ShardGroup.distributed([ctx], [full], rank, world, T, HostStagedDist(dist))
        res = []
        for t in range(T):
            K = cs.keep_count(0.05, P + t)
            qs = np.stack([q[P + t]] * group)
            with torch.cuda.stream(stream):
                out, sels = grp.decode_step(torch.from_numpy(qs).cuda(), torch.from_numpy(k[P + t][None]).cuda(),
                                            torch.from_numpy(v[P + t][None]).cuda(), want_selected=True, k_max=K)
                out = out.cpu().numpy()
            if rank == 0:
                ref = control.decode_step(qs, k[P + t], v[P + t])
                ref = ref if isinstance(ref, list) else [ref]
                res.append([(np.array_equal(sels[h], ref[h].selected), rel_err(out[h], ref[h].output))
                            for h in range(group)])
        if rank == 0:
            q_out.put(res)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_distributed_shard_group_two_ranks_one_gpu():
    """ShardGroup.distributed with world 2 (two processes on cuda:0, gloo with
    host-staged collectives): selections equal the unsharded session's exactly,
    outputs within 1e-3."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    P, T = 16384, 5
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, P, T, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    for t, heads in enumerate(res):
        for h, (same, err) in enumerate(heads):
            assert same, (t, h)
            assert err <= 1e-3, (t, h, err)
