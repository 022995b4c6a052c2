#!/usr/bin/env python
"""Benchmark of the CSAttention decode hot path on B200 (BASELINE.json metric).

Workload (default, --config c3): BASELINE config 3 — a Llama-3.1-8B-shaped
attention layer (32 query / 8 KV heads, d=128, GQA groups of 4) at 128K
prefill context, batch-16 decode sharing one prefilled context, CSAttention
defaults m=8, C=64, alpha=0.2, rho=0.05 (95% sparsity), R=32, tau=1.
Synthetic data from the reference generator: KV head g uses
spec {dim 128, clusters 8, seed mix_seed(2026, g)}, its 4 query heads use
dwell {32, 16, 64, 8}; the KV head's tables are built on the GPU (exact
k-means + top-L) over the 4 heads' pooled prefill queries; the 16 sequences
are forks of that prefill (reference value semantics), sequence s decoding
rows [P + s*T, P + (s+1)*T).

A step = one decode step of the whole layer for all 16 sequences: centroid
routing, gather/accumulate, top-K, sparse attention for 512 (sequence, query
head) problems, then append + streaming insert for 128 (sequence, KV head)
sessions: 2 kernel launches.

value = device time per layer-step in microseconds (lower is better), CUDA
events on the launching stream, max over ranks. e2e = the same through the
public C ABI with host (pinned) buffers, H2D of the step's q/k/v and D2H of
its outputs inside the timed region. Multi-GPU: KV heads are sharded across
ranks (rank r owns heads g with g % N == r), no data-path collective, so the
layer latency should fall with N ("strong" scaling).

--impl reference: the reference CPU implementation (oracle/_ref, built from the
unmodified sources) on the box's host cores: a bounded sample of the same
workload (one sequence, H KV heads built by the reference's own build_index,
one host thread per KV head), scaled to the full layer-step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (prefill P, sequences, layers, description)
    "c2": (32768, 1, 1, "Llama-3.1-8B-shaped attention layer (32 q / 8 KV heads, d=128) at 32K "
                        "context, 1 B200"),
    "c2o": (32768, 1, 1, "c2 in the CPU<->GPU offload mode: KV rows in pinned host memory, tables "
                         "in HBM; a step moves only the selected K/V rows over the host link"),
    "c3": (131072, 16, 1, "Llama-3.1-8B-shaped layer at 128K context, batch-16 decode sharing one "
                          "prefilled context"),
    "c4": (131072, 1, 32, "full 32-layer Llama-3.1-8B-shaped decode at 128K, KV heads sharded "
                          "across the GPUs of the run"),
    "c5": (1048576, 1, 1, "1M-token context, Llama-3.1-8B-shaped layer, sequence-sharded (>= 4 "
                          "shards, spread over the GPUs of the run) with the histogram / bucket / "
                          "LSE / victim collectives"),
}
N_KV, GROUP, D, M, C_CENT = 8, 4, 128, 8, 64
DWELLS = (32, 16, 64, 8)
METRIC = "decode-step sparse-attn latency (us) & HBM GB/s vs roofline, 128K ctx, 95% sparsity"


def mix_seed(seed: int, salt: int) -> int:
    """splitmix64 sub-seed (util.hpp:61-66)."""
    mask = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15 * (salt + 1)) & mask
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
    return z ^ (z >> 31)


def keep_count(rho: float, n: int) -> int:
    import math
    return max(1, int(math.ceil(rho * n - 1e-9)))


def gen_head(cs, g: int, rows: int):
    """Synthetic rows of KV head g: 4 query streams (dwells), keys, values."""
    seed = mix_seed(2026, g)
    qs = []
    k = v = None
    for dw in DWELLS:
        q, kk, vv = cs.make_synthetic(cs.SyntheticSpec(rows=rows, dim=D, clusters=8, seed=seed,
                                                       dwell=dw))
        qs.append(q)
        if k is None:
            k, v = kk, vv
    return np.stack(qs, 1), k, v  # q: [rows, 4, d]


def gen_heads(cs, heads, rows):
    with ThreadPoolExecutor(max_workers=min(16, 4 * len(heads))) as ex:
        return list(ex.map(lambda g: gen_head(cs, g, rows), heads))


class ClockSampler:
    """nvidia-smi-equivalent clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
            "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
            "display_clock_setting": 0x100,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in names.items():
                    if r & bit and n != "gpu_idle":
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str, config: str):
    """Per-launch DRAM bytes (read + write) of `kernel` from the committed ncu
    capture (profiles/ncu_<kernel>_<config>.json, one `ncu --set full` launch)."""
    p = os.path.join(ROOT, "profiles", f"ncu_{kernel}_{config}.json")
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


# --------------------------------------------------------------------------
# reference arm / cpu baseline
# --------------------------------------------------------------------------

def run_reference(args, P, n_seq, rank):
    """The reference CPU implementation on this host: bounded sample, scaled."""
    if rank != 0:
        return None
    import paper_2604_08584_b200 as cs  # host-side generator only (bit-identical)
    from oracle import bindings as ob
    if not ob.ref_available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libcsattn_ref.so not built"}
    cores = os.cpu_count() or 1
    H = max(1, min(N_KV, cores))
    steps, warm = args.steps, args.warmup
    T = steps + warm
    heads = list(range(H))
    data = gen_heads(cs, heads, P + T)
    widths = [D // M] * M
    rc = cs.RetrievalConfig()

    def build(g):
        q, k, v = data[g]
        pooled = np.ascontiguousarray(np.concatenate([q[:P, r] for r in range(GROUP)]))
        ic = cs.IndexConfig(alpha=0.2, centroids=C_CENT, seed=mix_seed(1, g), score_bits=32)
        return ob.RefSession.prefill(pooled, k[:P], v[:P], widths, ic, rc, GROUP)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=H) as ex:
        sess = list(ex.map(build, heads))
    build_s = time.perf_counter() - t0
    qs = np.stack([data[g][0][P:P + T] for g in heads])     # [H, T, 4, d]
    ks = np.stack([data[g][1][P:P + T] for g in heads])     # [H, T, d]
    vs = np.stack([data[g][2][P:P + T] for g in heads])
    ob.ref_bench(sess, qs[:, :warm], ks[:, :warm], vs[:, :warm], warm, H) if warm else None
    sec = ob.ref_bench(sess, qs[:, warm:], ks[:, warm:], vs[:, warm:], steps, H)
    per_step = sec / steps                                   # H KV heads in parallel
    sessions_total = N_KV * n_seq
    layer_us = per_step * (sessions_total / H) * 1e6
    sample = (f"1 sequence x {H} KV heads (group {GROUP}, {4 * H} query heads) at N={P}, "
              f"reference build_index ({build_s:.1f}s, untimed), {steps} timed steps on {H} "
              f"threads; scaled x{sessions_total / H:g} to the full layer-step")
    return {"layer_us": layer_us, "cores": H, "sample": sample, "kind": "reference",
            "per_kvhead_step_ms": per_step * 1e3}


def cpu_baseline_from_gpu(cs, ob, sessions_by_head, data, P, n_seq, steps, T_used):
    """cpu_baseline leg of our arm: the reference's decode path (oracle/_ref) on
    the tables the GPU built (bit-identical to build_index, tests/), one host
    thread per KV head, bounded sample of the same workload."""
    if not ob.ref_available():
        return None
    cores = os.cpu_count() or 1
    heads = sorted(sessions_by_head)[:max(1, min(len(sessions_by_head), cores))]
    widths = [D // M] * M
    rc = cs.RetrievalConfig()
    refs = []
    for g in heads:
        s = sessions_by_head[g]
        inf = s.info()
        lens, idx, sc, cent = s.export_index()
        q, k, v = data[g]
        kk, vv = s.read_kv(0, inf.context_len)
        refs.append(ob.RefSession.from_index(cent, lens, idx, sc, inf.list_capacity, inf.alpha,
                                             kk, vv, widths, rc, GROUP))
    # continue sequence 0 of each head from where the GPU left it
    base = P + T_used
    qs = np.stack([data[g][0][base:base + steps] for g in heads])
    ks = np.stack([data[g][1][base:base + steps] for g in heads])
    vs = np.stack([data[g][2][base:base + steps] for g in heads])
    sec = ob.ref_bench(refs, qs, ks, vs, steps, len(heads))
    per_step = sec / steps
    sessions_total = N_KV * n_seq
    return {"value": per_step * (sessions_total / len(heads)) * 1e6, "unit": "us",
            "cores": len(heads), "kind": "reference",
            "sample": (f"reference decode path (oracle/_ref) on the GPU-built tables of "
                       f"{len(heads)} KV heads x 1 sequence (group {GROUP}) at N~{base}, "
                       f"{steps} steps, one thread per KV head; scaled "
                       f"x{sessions_total / len(heads):g} to the full layer-step")}


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

def run_c5(args, config, P, rank, world, local):
    """Config c5: a 1M-token layer (8 KV heads x GQA 4), sequence-sharded.
    Shards are tile-aligned key ranges of <= 256K keys; there are
    max(4, world) of them, world/ranks each holding the same number. Every
    rank builds the 8 full sessions (deterministic: identical everywhere),
    keeps its shards and drops the rest. A step = one sharded decode step of
    the layer (ShardGroup.decode_step): per-shard scan, then the histogram
    all-reduce, bucket all-gather, count all-gather, attention-partial
    all-gather + LSE merge, victim all-reduce and the insert."""
    import torch
    import paper_2604_08584_b200 as cs
    from paper_2604_08584_b200.sharding import ShardGroup

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    n_total = max(4, world)
    L = n_total // world
    if L * world != n_total:
        raise SystemExit(f"c5 needs a world size dividing {n_total}")
    ctxs = [cs.Context(local, stream.cuda_stream) for _ in range(L)]
    steps, warm = args.steps, args.warmup
    e2e_steps = min(steps, 5)
    T = warm + steps + e2e_steps + 1
    widths = [D // M] * M
    rc = cs.RetrievalConfig()
    heads = list(range(N_KV))
    t0 = time.perf_counter()
    data = dict(zip(heads, gen_heads(cs, heads, P + T)))
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    full = []
    for g0 in range(0, len(heads), 4):  # 4 heads per csattn_prefill_batch (host RAM: pooled queries)
        hb = heads[g0:g0 + 4]
        rows_b = [(np.ascontiguousarray(np.concatenate([data[g][0][:P, r] for r in range(GROUP)])),
                   data[g][1][:P], data[g][2][:P]) for g in hb]
        ics = [cs.IndexConfig(alpha=0.2, centroids=C_CENT, seed=mix_seed(1, g), score_bits=32)
               for g in hb]
        full += cs.prefill_batch(ctxs[0], rows_b, widths, ics, rc, group=GROUP, max_decode_steps=1)
        del rows_b
    t_build = time.perf_counter() - t0
    if world == 1:
        grp = ShardGroup.local(ctxs, full, max_decode_steps=T)
    else:
        grp = ShardGroup.distributed(ctxs, full, rank, world, T, dist)
    for f in full:
        f.close()
    nq = N_KV * GROUP
    qh = np.stack([np.concatenate([data[g][0][P + t] for g in heads]) for t in range(T)])
    kh = np.stack([np.stack([data[g][1][P + t] for g in heads]) for t in range(T)])
    vh = np.stack([np.stack([data[g][2][P + t] for g in heads]) for t in range(T)])
    qd, kd, vd = (torch.from_numpy(x).cuda() for x in (qh, kh, vh))
    torch.cuda.synchronize()

    def step(t):
        with torch.cuda.stream(stream):
            return grp.decode_step(qd[t], kd[t], vd[t])

    t = 0
    for _ in range(warm):
        step(t)
        t += 1
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = P + t
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
        for _ in range(steps):
            step(t)
            t += 1
        with torch.cuda.stream(stream):
            ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if dist:
        tm = torch.tensor([ms], device="cuda")
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ms = float(tm.item())
    ms_per_step = ms / steps
    # e2e: host inputs copied in, output copied out, inside the timed region
    qp = torch.from_numpy(qh).pin_memory()
    kp = torch.from_numpy(kh).pin_memory()
    vp_ = torch.from_numpy(vh).pin_memory()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    te0 = time.perf_counter()
    for _ in range(e2e_steps):
        with torch.cuda.stream(stream):
            out, _ = grp.decode_step(qp[t].cuda(non_blocking=True), kp[t].cuda(non_blocking=True),
                                     vp_[t].cuda(non_blocking=True))
            host_out = out.cpu()
        t += 1
    e2e_ms = (time.perf_counter() - te0) * 1e3 / e2e_steps
    if dist:
        tm = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        e2e_ms = float(tm.item())
    assert np.isfinite(host_out.numpy()).all()
    L_list = 209716
    Kmean = keep_count(0.05, n0 + steps // 2)
    per_query = nq * (M * L_list * 8 + Kmean * (2 * D * 4 + 4) + C_CENT * D * 4 + 2 * D * 4)
    peak, peak_src = measured_peak()
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": ms_per_step * 1e3, "unit": "us", "n_gpus": world,
            "steps": steps, "warmup": warm, "ms_per_step": ms_per_step, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference make_synthetic, prefix-stable rows)",
            "config": dict(config, parallelism=f"sequence shards x{n_total} over {world} GPU(s)",
                           l2_policy="working set >> L2; no flush"),
            "hbm_gbs_per_step": per_query / (ms_per_step * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": "layer step (all sharded phases)",
                         "achieved": per_query / (ms_per_step * 1e-3) / 1e9, "peak": peak * world,
                         "unit": "GB/s", "frac": per_query / (ms_per_step * 1e-3) / 1e9 / (peak * world),
                         "traffic": None, "peak_source": peak_src,
                         "alg_bytes_per_launch": per_query, "alg_bytes": "per query head (8(d))"},
            "e2e": {"value": e2e_ms * 1e3, "unit": "us",
                    "h2d_bytes_per_step": int(qh[0].nbytes + kh[0].nbytes + vh[0].nbytes),
                    "d2h_bytes_per_step": int(nq * D * 4)},
            "gpu_launches": int(sum(c.launches for c in ctxs)),
            "clocks": clk.summary(),
            "setup_s": {"synthetic": round(t_gen, 2), "gpu_build": round(t_build, 2)},
            "cpu_baseline": None,
        }))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-steps", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    P, n_seq, n_layers, desc = CONFIGS[args.config]
    config = {"workload": f"{args.config}: {desc}", "prefill": P, "sequences": n_seq,
              "layers": n_layers,
              "kv_heads": N_KV, "q_heads": N_KV * GROUP, "d": D, "m": M, "C": C_CENT,
              "alpha": 0.2, "rho": 0.05, "window": 32, "tau": 1}

    if args.impl == "reference":
        res = run_reference(args, P, n_seq * n_layers, rank)
        if rank != 0:
            return
        if "unavailable" in res:
            print(json.dumps(res))
            return
        v = res["layer_us"]
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": "us", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v / 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference make_synthetic)", "config": config,
            "cpu_baseline": {"value": v, "unit": "us", "cores": res["cores"], "kind": "reference",
                             "sample": res["sample"]},
            "e2e": {"value": v, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    import torch
    import paper_2604_08584_b200 as cs
    from paper_2604_08584_b200 import _abi
    import ctypes as C

    if args.config == "c5":
        return run_c5(args, config, P, rank, world, local)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    ctx = cs.Context(local, stream.cuda_stream)
    if args.config == "c2o":  # offload mode
        ctx.set_kv_placement("host")
        config["kv_placement"] = "pinned host memory (mapped), tables in HBM"

    steps, warm = args.steps, args.warmup
    prof_steps = min(steps, 10)
    e2e_steps = min(steps, 10)
    graph_steps = min(steps, 10)
    T = warm + steps + prof_steps + e2e_steps + 3 * graph_steps + 2
    from paper_2604_08584_b200.sharding import kv_head_shard
    my_heads = kv_head_shard(N_KV, world, rank)
    widths = [D // M] * M
    rc = cs.RetrievalConfig()

    t0 = time.perf_counter()
    data = dict(zip(my_heads, gen_heads(cs, my_heads, P + n_layers * n_seq * T + args.cpu_steps)))
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    # the layer's KV heads in one csattn_prefill_batch (one k-means launch)
    rows_b = [(np.ascontiguousarray(np.concatenate([data[g][0][:P, r] for r in range(GROUP)])),
               data[g][1][:P], data[g][2][:P]) for g in my_heads]
    ics = [cs.IndexConfig(alpha=0.2, centroids=C_CENT, seed=mix_seed(1, g), score_bits=32)
           for g in my_heads]
    base_sessions = dict(zip(my_heads, cs.prefill_batch(ctx, rows_b, widths, ics, rc, group=GROUP,
                                                        max_decode_steps=T)))
    del rows_b
    t_build = time.perf_counter() - t0
    # Session order: layer-major, then KV head, then sequence. Sequence 0 of
    # layer 0 is the prefilled session; every other (layer, sequence) is a fork
    # of it (tables copied, prefill rows shared: c3's 16 sequences share one
    # prefill; c4's layers start from layer 0's tables, build time only), and
    # decodes its own rows of the head's stream, [P + (l*n_seq + s)*T, +T).
    t0 = time.perf_counter()
    sessions, rows = [], []
    for layer in range(n_layers):
        for g in my_heads:
            for s in range(n_seq):
                first = layer == 0 and s == 0
                sessions.append(base_sessions[g] if first else base_sessions[g].fork(T))
                rows.append((g, layer * n_seq + s))
    t_fork = time.perf_counter() - t0
    ns = len(sessions)
    nq = ns * GROUP
    ns_l = ns // n_layers  # sessions per layer (a layer = one decode_batch call)
    handles = [(C.c_void_p * ns_l)(*[s.h.value for s in sessions[l * ns_l:(l + 1) * ns_l]])
               for l in range(n_layers)]
    # per-step inputs for every session: q [T, ns*4, d], k/v [T, ns, d]
    qh = np.empty((T, nq, D), np.float32)
    kh = np.empty((T, ns, D), np.float32)
    vh = np.empty((T, ns, D), np.float32)
    for i, (g, s) in enumerate(rows):
        q, k, v = data[g]
        r0 = P + s * T
        qh[:, i * GROUP:(i + 1) * GROUP] = q[r0:r0 + T]
        kh[:, i] = k[r0:r0 + T]
        vh[:, i] = v[r0:r0 + T]
    qd = torch.from_numpy(qh).cuda()
    kd = torch.from_numpy(kh).cuda()
    vd = torch.from_numpy(vh).cuda()
    outd = torch.empty((T, nq, D), dtype=torch.float32, device="cuda")
    L = base_sessions[my_heads[0]].info().list_capacity
    torch.cuda.synchronize()
    lib = cs.lib()

    def step(t, flags=_abi.NO_SYNC, sel=None, sel_stride=0):
        # one decode step of the model slice: the layers in order, each one
        # csattn_decode_batch over its (KV head x sequence) sessions
        for l in range(n_layers):
            qs, ks = l * ns_l * GROUP, l * ns_l
            st = lib.csattn_decode_batch(
                ctx.h, ns_l, handles[l], C.c_void_p(qd[t, qs].data_ptr()),
                C.c_void_p(kd[t, ks].data_ptr()), C.c_void_p(vd[t, ks].data_ptr()),
                C.c_void_p(outd[t, qs].data_ptr()),
                None if sel is None else C.c_void_p(sel[qs].data_ptr()), sel_stride, flags)
            cs._check(st)

    # ---- warmup ----
    t = 0
    for _ in range(warm):
        step(t)
        t += 1
    ctx.synchronize()
    # ---- timed region (device time, CUDA events on the launching stream) ----
    launches0 = ctx.launches
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    n_at_start = P + t
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
        for _ in range(steps):
            step(t)
            t += 1
        with torch.cuda.stream(stream):
            ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    gpu_launches = ctx.launches - launches0
    ms = ev0.elapsed_time(ev1)
    if dist:
        tm = torch.tensor([ms], device="cuda")
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ms = float(tm.item())
        dist.barrier()
    ms_per_step = ms / steps
    # ---- per-kernel durations (separate pass, events around each launch) ----
    ctx.profile(True)
    n_prof0 = P + t
    for _ in range(prof_steps):
        step(t)
        t += 1
    prof = ctx.profile_read(reset=True)
    ctx.profile(False)
    nps = max(1, prof["steps"]) / n_layers  # profiled model steps (one call per layer)
    sel_ms = prof["select_ms"] / nps          # per model step: all layers' launches
    att_ms = prof["attend_ms"] / nps
    ins_ms = prof["insert_ms"] / nps
    # ---- algorithmic bytes ----
    # per query head ("per-query"): m*L gathered (u32, f32) entries + C*d*4
    # centroids + d*4 q + K*4 indices (select); K*(2*d*4 + 4) selected K/V rows
    # and indices + 2*d*4 q/out (attend). Unique (what one pass over HBM must
    # move): the union of the tables a session's query heads gather, and per KV
    # head the union of the selected prefill rows over its 64 (sequence, head)
    # problems (the 16 sequences share the prefill rows) plus each session's
    # own appended rows. Measured on the last profiled step (gather) and on one
    # extra step with the selected sets read back (attend).
    u_ent = C.c_uint64()
    t_ent = C.c_uint64()
    uniq_entries = tot_entries = 0
    for sh in sessions:
        cs._check(lib.csattn_session_gather_stats(sh.h, C.byref(u_ent), C.byref(t_ent)))
        uniq_entries += u_ent.value
        tot_entries += t_ent.value
    Kp = keep_count(0.05, n_prof0 + prof_steps - 1)
    sel_unique = (uniq_entries * 8 + ns * C_CENT * D * 4 + nq * (D * 4 + Kp * 4))
    sel_perq = (tot_entries * 8 + nq * (C_CENT * D * 4 + D * 4 + Kp * 4))
    maxK = keep_count(0.05, P + t)
    seld = torch.zeros((nq, maxK), dtype=torch.int32, device="cuda")
    step(t, flags=0, sel=seld, sel_stride=maxK)
    Ka = keep_count(0.05, P + t)
    t += 1
    selh = seld.cpu().numpy().astype(np.int64)[:, :Ka]
    uniq_rows = 0
    for l in range(n_layers):  # every layer's KV is its own memory in a real model
        for gi, g in enumerate(my_heads):
            b = (l * len(my_heads) + gi) * n_seq * GROUP
            rows_g = selh[b:b + n_seq * GROUP]
            uniq_rows += np.unique(rows_g[rows_g < P]).size
            for sidx in range(n_seq):  # appended rows are per session
                r = rows_g[sidx * GROUP:(sidx + 1) * GROUP]
                uniq_rows += np.unique(r[r >= P]).size
    att_unique = uniq_rows * 2 * D * 4 + nq * (Ka * 4 + 2 * D * 4)
    att_perq = nq * (Ka * (2 * D * 4 + 4) + 2 * D * 4)
    peak, peak_src = measured_peak()
    kernels = {
        "select": {"ms": sel_ms, "alg_bytes_unique": sel_unique, "alg_bytes_per_query": sel_perq,
                   "gbs": sel_unique / (sel_ms * 1e-3) / 1e9},
        "attend": {"ms": att_ms, "alg_bytes_unique": att_unique, "alg_bytes_per_query": att_perq,
                   "gbs": att_unique / (att_ms * 1e-3) / 1e9},
        "insert": {"ms": ins_ms},
    }
    for v in kernels.values():
        if "gbs" in v:
            v["frac"] = v["gbs"] / peak
    dom = "select" if sel_ms >= att_ms else "attend"
    dec_ms = kernels[dom]["ms"]
    alg_bytes = kernels[dom]["alg_bytes_unique"]
    achieved = kernels[dom]["gbs"]
    step_bytes = sel_unique + att_unique
    # ---- e2e: public API with pinned host buffers, copies inside the timed region ----
    qp = torch.from_numpy(qh).pin_memory()
    kp = torch.from_numpy(kh).pin_memory()
    vp_ = torch.from_numpy(vh).pin_memory()
    op = torch.empty((T, nq, D), dtype=torch.float32).pin_memory()
    ctx.synchronize()
    if dist:
        dist.barrier()
    te0 = time.perf_counter()
    for _ in range(e2e_steps):
        for l in range(n_layers):
            qs, ks = l * ns_l * GROUP, l * ns_l
            st = lib.csattn_decode_batch(ctx.h, ns_l, handles[l], C.c_void_p(qp[t, qs].data_ptr()),
                                         C.c_void_p(kp[t, ks].data_ptr()),
                                         C.c_void_p(vp_[t, ks].data_ptr()),
                                         C.c_void_p(op[t, qs].data_ptr()), None, 0,
                                         _abi.HOST_BUFFERS)
            cs._check(st)
        t += 1
    e2e_ms = (time.perf_counter() - te0) * 1e3 / e2e_steps
    if dist:
        tm = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        e2e_ms = float(tm.item())
    assert np.isfinite(op[t - 1].numpy()).all()
    assert torch.isfinite(outd[warm:warm + steps]).all()
    # ---- whole-run CUDA graph (csattn_decode_run): graph_steps
    # steps per call, capture + instantiate + launch + sync inside the clock;
    # once from device buffers, once from pinned host buffers (all steps' inputs
    # copied in and outputs out inside the call) ----
    graph = {"steps_per_call": graph_steps}
    for mode in ("warmup", "device", "e2e"):  # warmup: first-call arena / staging growth
        hostb = mode != "device"
        src = (qp, kp, vp_) if hostb else (qd, kd, vd)
        bufs = []
        for l in range(n_layers):
            qs, ks = l * ns_l * GROUP, l * ns_l
            sl = [x[t:t + graph_steps, a:a + n].contiguous() for x, a, n in
                  zip(src, (qs, ks, ks), (ns_l * GROUP, ns_l, ns_l))]
            if hostb:
                sl = [x.pin_memory() for x in sl]
            o = torch.empty((graph_steps, ns_l * GROUP, D), dtype=torch.float32,
                            device="cpu" if hostb else "cuda")
            bufs.append(sl + [o.pin_memory() if hostb else o])
        torch.cuda.synchronize()
        ctx.synchronize()
        if dist:
            dist.barrier()
        tg0 = time.perf_counter()
        for l in range(n_layers):
            gq, gk, gv, go = bufs[l]
            cs._check(lib.csattn_decode_run(
                ctx.h, ns_l, handles[l], graph_steps, C.c_void_p(gq.data_ptr()),
                C.c_void_p(gk.data_ptr()), C.c_void_p(gv.data_ptr()), C.c_void_p(go.data_ptr()),
                None, 0, None, _abi.HOST_BUFFERS if hostb else 0))
        g_ms = (time.perf_counter() - tg0) * 1e3 / graph_steps
        if dist:
            tm = torch.tensor([g_ms], device="cuda")
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            g_ms = float(tm.item())
        if mode != "warmup":
            graph[f"{mode}_us_per_step"] = g_ms * 1e3
        assert all(torch.isfinite(b[3]).all() for b in bufs)
        t += graph_steps

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import bindings as ob
            cpu = cpu_baseline_from_gpu(cs, ob, base_sessions, data, P, n_seq * n_layers,
                                        args.cpu_steps, t)
        except Exception as e:  # reported, never fatal for the GPU number
            cpu = {"value": None, "error": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": ms_per_step * 1e3,
            "unit": "us",
            "n_gpus": world,
            "steps": steps,
            "warmup": warm,
            "ms_per_step": ms_per_step,
            "higher_is_better": False,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (reference make_synthetic, prefix-stable rows)",
            "config": dict(config, parallelism=f"kv-head shard x{world}", l2_policy=(
                "working set (tables ~14 GB + KV 1 GB per GPU at c3) >> 126 MB L2; no flush")),
            "hbm_gbs_per_step": step_bytes / (ms_per_step * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": f"csa::{dom}_kernel", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": ncu_traffic(dom, args.config), "peak_source": peak_src,
                         "alg_bytes_per_launch": alg_bytes, "alg_bytes": "unique (SURVEY 8(d))",
                         "kernel_ms": dec_ms, "problems_per_launch": nq, "kernels": kernels},
            "e2e": {"value": e2e_ms * 1e3, "unit": "us",
                    "h2d_bytes_per_step": int(qh[0].nbytes + kh[0].nbytes + vh[0].nbytes),
                    "d2h_bytes_per_step": int(op[0].numel() * 4)},
            "graph": graph,
            "gpu_launches": int(gpu_launches),
            "clocks": clk.summary(),
            "setup_s": {"synthetic": round(t_gen, 2), "gpu_build": round(t_build, 2),
                        "fork": round(t_fork, 2)},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
