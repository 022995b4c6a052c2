"""KV-head sharding of a CSAttention layer across the GPUs of one box
(SURVEY.md §8(e), config c4): rank r owns the KV heads g with g % world == r,
their GQA query heads, tables, KV rows and forks. Build and decode are local;
the only exchange is the optional output gather (32 x 128 x 4 B = 16 KB per
layer step), done here with one all_gather over the process group.
"""
from __future__ import annotations

import ctypes as C

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


# ---------------------------------------------------------------------------
# Sequence sharding: one logical KV-head session
# split by key range over shards; the decode step runs the C ABI's phases
# (csattn_shard_step) with the collectives between them. Two transports:
#   local  all shards in this process (one context each, same device or
#          several): collectives are plain tensor ops;
#   dist   one shard per rank (torch.distributed, NCCL): all_reduce /
#          all_gather on the same buffers.
# The union of the shards' selections equals the unsharded selection (tests).
# ---------------------------------------------------------------------------
SHARD_ALIGN = 4096  # select tile: shard boundaries are multiples of it

_U64_FLIP = -(1 << 63)  # uint64 <-> order-preserving int64 (XOR the sign bit)


def shard_bounds(P: int, n_shards: int) -> list[tuple[int, int]]:
    """Key ranges [lo, hi) of the shards: tile-aligned, ascending; the last
    shard (the owner of appended keys) ends at P."""
    tiles = -(-P // SHARD_ALIGN)
    if n_shards < 1 or n_shards > tiles:
        raise ValueError(f"{n_shards} shards for {tiles} tiles")
    cuts = [(tiles * j) // n_shards * SHARD_ALIGN for j in range(n_shards)] + [P]
    return [(cuts[j], cuts[j + 1]) for j in range(n_shards)]


def coll_all_reduce_sum(bufs, dist=None):
    """In place: every local buffer becomes the sum over all shards (local
    ones, then across ranks)."""
    import torch
    tot = torch.stack(bufs).sum(0) if len(bufs) > 1 else bufs[0].clone()
    if dist is not None:
        dist.all_reduce(tot)
    for b in bufs:
        b.copy_(tot)


def coll_all_gather(bufs, dist=None, world=1):
    """[n_shards, ...]: every shard's buffer in global shard order (rank-major,
    then local order)."""
    import torch
    mine = torch.stack(bufs).contiguous()
    if dist is None:
        return mine
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    return torch.cat(parts).contiguous()


def coll_all_reduce_min_u64(bufs, dist=None):
    """In place: elementwise min of uint64 values stored in int64 tensors
    (sign bit flipped so that signed order equals unsigned order)."""
    import torch
    m = (torch.stack(bufs) ^ _U64_FLIP).min(0).values
    if dist is not None:
        dist.all_reduce(m, op=dist.ReduceOp.MIN)
    m = m ^ _U64_FLIP
    for b in bufs:
        b.copy_(m)


class HostStagedDist:
    """torch.distributed with every collective staged through host memory:
    for a transport without device tensors (gloo), or several ranks on one GPU
    (NCCL refuses two ranks on the same device). Same calls as the subset of
    torch.distributed that ShardGroup uses."""

    def __init__(self, dist):
        self.d = dist
        self.ReduceOp = dist.ReduceOp

    def all_reduce(self, t, op=None):
        h = t.cpu()
        self.d.all_reduce(h, op=self.d.ReduceOp.SUM if op is None else op)
        t.copy_(h)

    def all_gather(self, parts, t):
        hp = [p.cpu() for p in parts]
        self.d.all_gather(hp, t.cpu())
        for p, h in zip(parts, hp):
            p.copy_(h)


class ShardGroup:
    """Sharded decode of a set of KV-head sessions.

    local: ShardGroup.local(contexts, full_sessions, max_decode_steps) —
           contexts[j] holds shard j of every session.
    dist:  ShardGroup.distributed(ctx, full_sessions, rank, world, ...) —
           this rank holds shard `rank`; collectives over the default group.
    decode_step(q, new_keys, new_values) takes device tensors (sum of groups
    x d, n x d, n x d) and returns the output (sum of groups x d) and, if
    asked, each query head's selected key indices (ascending).
    """

    def __init__(self, ctxs, shard_sessions, bounds, dist=None, rank=0, world=1):
        import torch
        from . import _abi, lib
        self.torch, self._abi, self.lib = torch, _abi, lib()
        self.ctxs = ctxs                # per local shard
        self.shards = shard_sessions    # [local shard][session]
        self.bounds = bounds            # all shards, global order
        self.dist, self.rank, self.world = dist, rank, world
        self.n_shards = len(bounds)
        self.first = rank * len(shard_sessions)  # global index of local shard 0
        s0 = shard_sessions[0][0]
        info = s0.info()
        self.d, self.groups = info.dim, [s.info().group for s in shard_sessions[0]]
        self.nq, self.ns = sum(self.groups), len(shard_sessions[0])
        hw, bw, pf, vw = (C.c_uint64() for _ in range(4))
        from . import _check
        self._check = _check
        _check(self.lib.csattn_shard_buffer_words(s0.h, C.byref(hw), C.byref(bw), C.byref(pf),
                                                  C.byref(vw)))
        self.hw, self.bw, self.pf, self.vw = hw.value, bw.value, pf.value, vw.value

    # -- construction --
    @classmethod
    def local(cls, ctxs, full_sessions, max_decode_steps):
        from . import Session, _check, lib
        P = full_sessions[0].info().prefill_len
        bounds = shard_bounds(P, len(ctxs))
        shards = []
        for j, (c, (lo, hi)) in enumerate(zip(ctxs, bounds)):
            row = []
            for fs in full_sessions:
                h = C.c_void_p()
                _check(lib().csattn_shard_create(c.h, fs.h, lo, hi, int(j == len(bounds) - 1),
                                                 max_decode_steps, C.byref(h)))
                row.append(Session(c, h))
            shards.append(row)
        return cls(ctxs, shards, bounds)

    @classmethod
    def distributed(cls, ctxs, full_sessions, rank, world, max_decode_steps, dist):
        """This rank holds shards [rank*len(ctxs), (rank+1)*len(ctxs)) of
        world*len(ctxs) shards (one context each, on this rank's GPU)."""
        from . import Session, _check, lib
        P = full_sessions[0].info().prefill_len
        L = len(ctxs)
        bounds = shard_bounds(P, world * L)
        shards = []
        for j, c in enumerate(ctxs):
            g = rank * L + j
            lo, hi = bounds[g]
            row = []
            for fs in full_sessions:
                h = C.c_void_p()
                _check(lib().csattn_shard_create(c.h, fs.h, lo, hi, int(g == len(bounds) - 1),
                                                 max_decode_steps, C.byref(h)))
                row.append(Session(c, h))
            shards.append(row)
        return cls(ctxs, shards, bounds, dist=dist, rank=rank, world=world)

    # -- one decode step --
    def _buffers(self, dev, want_selected, k_max):
        """Per-local-shard I/O buffers and ShardIoC structs, cached across steps
        (re-made only when the selected-set capacity grows)."""
        torch = self.torch
        key = (str(dev), bool(want_selected), int(k_max or 0))
        if getattr(self, "_cache_key", None) == key:
            return self._bufs, self._io
        nq, d = self.nq, self.d
        bufs, io = [], []
        for j in range(len(self.shards)):
            b = {
                "ghist": torch.zeros((nq, self.hw), dtype=torch.int32, device=dev),
                "bucket": torch.zeros((nq, self.bw), dtype=torch.int32, device=dev),
                "counts": torch.zeros((nq, 2), dtype=torch.int32, device=dev),
                "partial": torch.zeros((nq, self.pf), dtype=torch.float32, device=dev),
                "victim": torch.zeros((self.ns, self.vw), dtype=torch.int64, device=dev),
                "out": torch.empty((nq, d), dtype=torch.float32, device=dev),
                "nsel": torch.zeros((nq,), dtype=torch.int32, device=dev),
                "fail": torch.zeros((1,), dtype=torch.int32, device=dev),
            }
            if want_selected:
                b["sel"] = torch.zeros((nq, k_max), dtype=torch.int32, device=dev)
            bufs.append(b)
            x = self._abi.ShardIoC()
            x.ghist, x.bucket = b["ghist"].data_ptr(), b["bucket"].data_ptr()
            x.counts, x.partial = b["counts"].data_ptr(), b["partial"].data_ptr()
            x.out, x.victim = b["out"].data_ptr(), b["victim"].data_ptr()
            x.n_selected = b["nsel"].data_ptr()
            x.spec_fail = b["fail"].data_ptr()
            if want_selected:
                x.selected, x.sel_stride = b["sel"].data_ptr(), k_max
            x.shard_index = self.first + j
            x.n_shards = self.n_shards
            io.append(x)
        self._hs = [(C.c_void_p * self.ns)(*[s.h.value for s in row]) for row in self.shards]
        self._cache_key, self._bufs, self._io = key, bufs, io
        return bufs, io

    def decode_step(self, q, new_keys, new_values, want_selected=False, k_max=None):
        torch = self.torch
        dev = q.device
        L = len(self.shards)  # shards held by this process
        nq = self.nq
        bufs, io = self._buffers(dev, want_selected, k_max)
        for x in io:
            x.q, x.new_keys, x.new_values = q.data_ptr(), new_keys.data_ptr(), new_values.data_ptr()

        def run(phase):
            for j in range(L):
                self._check(self.lib.csattn_shard_step(self.ctxs[j].h, self.ns, self._hs[j], phase,
                                                       C.byref(io[j])))

        def all_reduce_sum(key):
            coll_all_reduce_sum([bb[key] for bb in bufs], self.dist)

        def all_gather(key, all_key):
            g = coll_all_gather([bb[key] for bb in bufs], self.dist, self.world)
            for j in range(L):
                bufs[j][all_key] = g
                setattr(io[j], all_key, g.data_ptr())

        def all_reduce_min_u64(key):
            coll_all_reduce_min_u64([bb[key] for bb in bufs], self.dist)

        A = self._abi
        import os
        prof = os.environ.get("CSATTN_SHARD_PROF")  # diagnostics: per-phase CUDA events
        marks = []

        def mark(name):
            if prof:
                e = torch.cuda.Event(enable_timing=True)
                e.record(torch.cuda.current_stream(dev))
                marks.append((name, e))
        mark("start")
        for bb in bufs:
            bb["fail"].zero_()
        run(A.SHARD_SCAN)
        mark("scan")
        all_reduce_sum("ghist")
        mark("ghist")
        run(A.SHARD_BUCKET)
        mark("bucket")
        # Did the speculative cut (previous step's threshold) miss on some query
        # head? The flag goes to pinned host memory asynchronously and is read
        # once MERGE is queued, so the host never waits mid-step. On a miss
        # every shard saw the same global histogram: rescan without speculation
        # and redo bucket..merge (mark clears its bitmap, emit/merge overwrite
        # their outputs; nothing persistent changes before INSERT).
        fail = torch.stack([bb["fail"] for bb in bufs]).max()
        if self.dist is not None:
            self.dist.all_reduce(fail, op=self.dist.ReduceOp.MAX)
        if getattr(self, "_fail_host", None) is None:
            self._fail_host = torch.zeros((1,), dtype=fail.dtype, pin_memory=True)
        self._fail_host.copy_(fail.reshape(1), non_blocking=True)
        fail_ev = torch.cuda.Event()
        fail_ev.record(torch.cuda.current_stream(dev))

        def select_tail():
            all_gather("bucket", "bucket_all")
            run(A.SHARD_MARK)
            mark("mark")
            all_gather("counts", "counts_all")
            run(A.SHARD_EMIT)
            mark("emit")
            all_gather("partial", "partial_all")
            run(A.SHARD_MERGE)
            mark("merge")
        select_tail()
        fail_ev.synchronize()
        if int(self._fail_host[0]):
            self.rescans = getattr(self, "rescans", 0) + 1
            for bb in bufs:
                bb["fail"].zero_()
            run(A.SHARD_RESCAN)
            all_reduce_sum("ghist")
            run(A.SHARD_BUCKET)
            select_tail()
        run(A.SHARD_VICTIM)
        all_reduce_min_u64("victim")
        run(A.SHARD_INSERT)
        mark("insert")
        if prof:
            marks[-1][1].synchronize()
            acc = getattr(self, "_prof", {})
            for (_, a), (n, b) in zip(marks, marks[1:]):
                acc[n] = acc.get(n, 0.0) + a.elapsed_time(b)
            acc["_steps"] = acc.get("_steps", 0) + 1
            self._prof = acc
            if acc["_steps"] % 8 == 0:
                import sys
                print("[shard prof] ms/step: " + ", ".join(
                    f"{k} {v / acc['_steps']:.3f}" for k, v in acc.items() if k != "_steps"),
                    file=sys.stderr)
        out = bufs[0]["out"]
        if not want_selected:
            return out, None
        # every shard's ascending local selection, concatenated in shard order
        n_all = coll_all_gather([bb["nsel"] for bb in bufs], self.dist, self.world).cpu().numpy()
        s_all = coll_all_gather([bb["sel"] for bb in bufs], self.dist, self.world).cpu().numpy()
        sels = []
        for p in range(nq):
            sels.append(np.concatenate([s_all[j][p, :n_all[j][p]] for j in range(self.n_shards)])
                        .astype(np.uint32))
        return out, sels
