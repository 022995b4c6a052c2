"""KV-head sharding host logic on CPU with gloo, world size 2:
each rank decodes only its KV heads (CPU oracle as the stand-in compute: this is
a host-logic test), the layer output is assembled by one all_gather, and must
equal the single-process layer output head for head."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2604_08584_b200 as cs
from paper_2604_08584_b200.sharding import gather_layer_output, kv_head_shard, shard_table

N_KV, GROUP, D, M, P, T = 4, 2, 32, 4, 256, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layer_outputs(heads):
    """[T, len(heads)*GROUP, D] outputs of a toy layer, computed by the CPU oracle."""
    from oracle import bindings as ob
    outs = np.zeros((T, len(heads) * GROUP, D), np.float32)
    for i, g in enumerate(heads):
        q, k, v = cs.make_synthetic(cs.SyntheticSpec(rows=P + T, dim=D, clusters=4, seed=100 + g))
        pooled = np.ascontiguousarray(np.concatenate([q[:P]] * GROUP))
        s = ob.OraSession.prefill(pooled, k[:P], v[:P], cs.uniform_widths(D, M),
                                  cs.IndexConfig(centroids=8, seed=1, score_bits=32),
                                  cs.RetrievalConfig(keep_ratio=0.1, recent_window=4), GROUP)
        for t in range(T):
            res = s.step(np.stack([q[P + t]] * GROUP), k[P + t], v[P + t])
            for h, (_, out, _, _) in enumerate(res):
                outs[t, i * GROUP + h] = out
    return outs


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = kv_head_shard(N_KV, world, rank)
    local = torch.from_numpy(_layer_outputs(mine))
    full = gather_layer_output(local, N_KV, GROUP, world, rank)
    if rank == 0:
        q.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_assignment_partitions_heads():
    for world in (1, 2, 4, 8):
        owned = [kv_head_shard(8, world, r) for r in range(world)]
        flat = sorted(g for o in owned for g in o)
        assert flat == list(range(8))
        assert all(len(o) == 8 // world for o in owned)
        assert shard_table(8, world).tolist() == [g % world for g in range(8)]
    with pytest.raises(ValueError):
        kv_head_shard(8, 2, 2)


def test_gloo_world2_output_gather_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = _layer_outputs(list(range(N_KV)))
    assert np.array_equal(full, ref)


def _coll_worker(rank, world, port, q):
    import paper_2604_08584_b200.sharding as sh
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = 2  # local shards per rank
    g = [torch.full((3, 4), 10 * rank + j, dtype=torch.int32) for j in range(L)]
    sh.coll_all_reduce_sum(g, dist)
    gathered = sh.coll_all_gather([torch.full((2,), 10 * rank + j) for j in range(L)], dist, world)
    big = (1 << 63) + 5  # uint64 values above 2^63, stored as int64
    v = [torch.tensor([(big + 100 * rank + 7 * j) - (1 << 64), rank + j], dtype=torch.int64)
         for j in range(L)]
    sh.coll_all_reduce_min_u64(v, dist)
    if rank == 0:
        q.put((g[0].tolist(), g[1].tolist(), gathered.tolist(), v[0].tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_shard_collectives():
    """The sequence-sharding collectives over ranks x local shards equal their
    single-process meaning: sum over all shards, gather in global shard order
    (rank-major), unsigned-64-bit min."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_coll_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    g0, g1, gathered, vmin = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    total = 0 + 1 + 10 + 11
    assert g0 == g1 == [[total] * 4] * 3
    assert gathered == [[0, 0], [1, 1], [10, 10], [11, 11]]
    assert vmin[0] == ((1 << 63) + 5) - (1 << 64) and vmin[1] == 0
