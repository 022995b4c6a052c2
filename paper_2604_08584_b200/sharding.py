"""KV-head sharding of a CSAttention layer across the GPUs of one box
(SURVEY.md §8(e), config c4): rank r owns the KV heads g with g % world == r,
their GQA query heads, tables, KV rows and forks. Build and decode are local;
the only exchange is the optional output gather (32 x 128 x 4 B = 16 KB per
layer step), done here with one all_gather over the process group.
"""
from __future__ import annotations

import numpy as np


def kv_head_shard(n_kv_heads: int, world: int, rank: int) -> list[int]:
    """KV heads owned by `rank` (round-robin, so 8 heads split evenly for
    world in {1, 2, 4, 8})."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return [g for g in range(n_kv_heads) if g % world == rank]


def gather_layer_output(local_out, n_kv_heads: int, group: int, world: int, rank: int,
                        dist=None):
    """Assemble the full layer output [n_seq, n_kv_heads*group, d] from each
    rank's [n_seq, len(own heads)*group, d] block (head-major within a rank,
    as bench.py orders its sessions). `local_out` is a torch tensor; with
    world == 1 it is returned unchanged."""
    import torch

    if world == 1:
        return local_out
    dist = dist or torch.distributed
    mine = kv_head_shard(n_kv_heads, world, rank)
    n_seq, _, d = local_out.shape
    # pad every rank's block to the largest shard so all_gather sees equal sizes
    cap = max(len(kv_head_shard(n_kv_heads, world, r)) for r in range(world)) * group
    buf = local_out.new_zeros((n_seq, cap, d))
    buf[:, :len(mine) * group] = local_out
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    full = local_out.new_empty((n_seq, n_kv_heads * group, d))
    for r in range(world):
        for i, g in enumerate(kv_head_shard(n_kv_heads, world, r)):
            full[:, g * group:(g + 1) * group] = parts[r][:, i * group:(i + 1) * group]
    return full


def shard_table(n_kv_heads: int, world: int) -> np.ndarray:
    """owner[g] = rank owning KV head g."""
    return np.array([g % world for g in range(n_kv_heads)], np.int64)
