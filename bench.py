#!/usr/bin/env python3
"""Bench: split-KV paged decode attention step (BASELINE configs[1]) on B200.

One "step" = one decode-attention layer step for a 64-request batch:
64 requests, KV lengths uniform_int(mt19937_64(0), 1024, 32768) (sum 1,068,741
tokens), GQA 32 q / 8 kv heads, head_dim 128, bf16 paged KV (page 16), i.e.
K1+K9 over ~4.38 GB of resident KV.  Metric: decode tok/s (requests decoded
per second through one attention layer) with the kernel's HBM GB/s vs the
measured peak in the roofline object.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU): the real DCP decode step across the
GPUs (bench_multi.py: K2 -> K1 -> K3 attention exchange + K4/K5 MoE
dispatch/combine over CUDA-IPC peer pools, weak scaling, value = whole-job
tok/s over max-over-ranks device time).  --replicas keeps the old mode: N
independent cfg2 replicas.
--impl reference: the reference's own CPU implementation
(dcpsim::sharded_attention_merge compiled from /root/reference sources into
oracle/_ref) timed on the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HQ, HKV, D, PAGE = 32, 8, 128, 16
METRIC = ("decode tok/s per attention layer (split-KV paged decode attention step, cfg2: 64 req, KV 1K-32K, "
          "GQA 32q/8kv, d128, bf16 paged)")
UNIT = "tok/s"
METRIC_MULTI = ("decode tok/s (DCP decode step on N GPUs: K2 -> K1 -> K3 attention exchange + K4/K5 MoE "
                "dispatch/combine, per attention+MoE layer)")
WORKLOAD = "cfg2 single-GPU split-KV decode attention: 64 requests, KV len uniform_int(mt19937_64(0),1024,32768) sum=1068741, GQA 32q/8kv, d=128, bf16 paged KV page=16"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """Samples SM clock + throttle reasons via NVML during the timed region."""

    def __init__(self, device: int):
        self.device, self.samples, self.reasons = device, [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    _NAMES = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._NAMES.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def _max_over_ranks(x, ws, device):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ CPU reference
def _tiled(n, seed, block=1 << 24):
    """n fp32 values: a seeded N(0,1) block of 64 MB (> L3) repeated; the reference's work is
    independent of the values, so only the footprint matters."""
    rng = np.random.default_rng(seed)
    return np.resize(rng.standard_normal(min(n, block), dtype=np.float32), n)


def cpu_reference_sample(steps: int, warmup: int = 0, token_budget: int | None = None, threads: int = 0):
    """Time dcpsim::sharded_attention_merge (the reference compiled from its sources, oracle/_ref)
    on the cfg2 step: all 64 requests (or the first requests up to token_budget), fp32, one
    shard per request, outer OpenMP over (request, q-head) on all host threads (BASELINE.md
    §4.3).  Returns (tok/s of the full cfg2 step, info)."""
    from tests import oracle_lib
    from paper_2605_21100_b200 import workload
    L = oracle_lib.reference()
    kind = "reference"
    if L is None:
        raise RuntimeError("oracle/_ref/libdcpsim_ref.so missing (build with make -C oracle)")
    lens = workload.cfg2_lengths()
    n = len(lens)
    if token_budget is not None:
        n, tot = 0, 0
        while n < len(lens) and tot < token_budget:
            tot += lens[n]
            n += 1
    sl = np.array(lens[:n], np.int64)
    q = np.random.default_rng(0).standard_normal((n, HQ, D), dtype=np.float32)
    kv_off = np.zeros(n, np.int64)
    kv_off[1:] = np.cumsum(sl[:-1] * HKV * D)
    kv_elems = int(sl.sum()) * HKV * D
    k = _tiled(kv_elems, 1)
    v = _tiled(kv_elems, 2)
    bounds = sl.copy()                       # one shard per request (CP = 1 on one GPU)
    bounds_off = np.arange(n, dtype=np.int64)
    nb = np.ones(n, np.int32)
    out = np.zeros((n, HQ, D), np.float32)
    th = threads or os.cpu_count() or 1
    P = oracle_lib.P
    times = []
    for i in range(warmup + max(steps, 1)):
        t0 = time.perf_counter()
        rc = L.dcpref_batch_decode_attn_f32(n, HQ, HKV, D, 1.0 / math.sqrt(D), P(q), P(k), P(v),
                                            P(kv_off), P(sl), P(bounds), P(bounds_off), P(nb), P(out), th)
        if i >= warmup:
            times.append(time.perf_counter() - t0)
        assert rc == 0
    full_tokens = sum(lens)
    full = n == len(lens)
    per_step = float(np.mean(times)) * (1.0 if full else full_tokens / float(sl.sum()))
    what = ("all 64 cfg2 requests" if full else
            f"first {n} of 64 cfg2 requests ({int(sl.sum())} of {full_tokens} KV tokens), scaled by token ratio")
    info = {"kind": kind, "cores": th,
            "sample": f"{what}: {int(sl.sum())} KV tokens, fp32, one shard each, mean of {len(times)} steps "
                      f"after {warmup} warm-up",
            "sample_s": float(np.mean(times)), "same_config": full}
    return 64.0 / per_step, info


# ------------------------------------------------------------------ planner path
PLANNER_SCENARIO = ("SURVEY §3.1: 1 node x 8 instances, gen_trace(seed 3, 1% long) — 2,336 active requests "
                    "then one DCP round admitting 64 new (Scheduler::step) + build_binding_config / "
                    "derive_routing_tables over the 2,400 actives")


def _planner_trace():
    from paper_2605_21100_b200 import workload
    tr = workload.gen_trace(3, 0.01, 240.0, 10.0, poisson=False)[:2400]
    return [(r[0], r[2]) for r in tr]


def planner_device(ctx):
    """K6 + K7 on the device for PLANNER_SCENARIO (CUDA events): the 2,336-admission round,
    the 64-admission round (which also rebalances the 2,336 actives), and K7 routing."""
    import torch
    from paper_2605_21100_b200.planner import DevicePlanner
    tr = _planner_trace()
    cap = 1 << 21
    times = []
    for rep in range(3):
        pl = DevicePlanner(ctx, 1, 8, 16, cap, "dcp", None, max_requests=4096, reserve_pages=8)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        pl.enqueue_many([r[0] for r in tr[:2336]], [r[1] for r in tr[:2336]])
        torch.cuda.synchronize()
        e[0].record()
        pl.step_async()
        e[1].record()
        assert len(pl.step_result()["committed"]) == 2336
        pl.enqueue_many([r[0] for r in tr[2336:]], [r[1] for r in tr[2336:]])
        torch.cuda.synchronize()
        e[2].record()
        pl.step_async()
        e[3].record()
        pl.build_routing()
        e[4].record()
        r = pl.step_result()
        torch.cuda.synchronize()
        assert len(r["committed"]) == 64
        times.append((e[2].elapsed_time(e[3]) * 1e3, e[3].elapsed_time(e[4]) * 1e3, e[0].elapsed_time(e[1]) * 1e3))
        pl.close()
    best = [min(t[i] for t in times) for i in range(3)]
    return {"device_step_us": best[0], "device_routing_us": best[1], "device_admit_2336_us": best[2]}


def planner_cpu_reference():
    """The same rounds through the reference (oracle/_ref, one host thread): Scheduler::step for
    the 2,336- and the 64-admission rounds, and build_binding_config + derive_routing_tables
    alone (no CSV writer)."""
    from tests import oracle_lib
    L = oracle_lib.reference()
    tr = _planner_trace()
    best_a, best_s, best_r = 1e9, 1e9, 1e9
    for rep in range(3):
        w = oracle_lib.World(L, "dcpref_", 1, 8, 16, 1 << 21, "dcp")
        for rid, ln in tr[:2336]:
            w.enqueue(rid, ln)
        t0 = time.perf_counter()
        assert len(w.step()["committed"]) == 2336
        t1 = time.perf_counter()
        for rid, ln in tr[2336:]:
            w.enqueue(rid, ln)
        t2 = time.perf_counter()
        r = w.step()
        t3 = time.perf_counter()
        assert len(r["committed"]) == 64
        best_a, best_s = min(best_a, t1 - t0), min(best_s, t3 - t2)
        best_r = min(best_r, w.time_routing_ns(5) * 1e-9)
    return {"cpu_reference_admit_2336_us": best_a * 1e6, "cpu_reference_step_us": best_s * 1e6,
            "cpu_reference_routing_us": best_r * 1e6, "cores": 1}


def _host_ram_ok(gb):
    try:
        import psutil
        return psutil.virtual_memory().available > gb * 1e9
    except Exception:
        return True


def cpu_reference_multi(ws: int, steps: int, warmup: int, token_budget: int | None = None, threads: int = 0):
    """The N > 1 arm's workload (bench_multi.py: one node of `ws` instances, 64 x 2,048 tokens per
    instance + ws-1 x 131,073 per node, then the cfg4 MoE exchange with identity experts) through
    the reference on the host cores: its Scheduler::step places every request (kv binding and
    splits), then per step dcpsim::sharded_attention_merge of every request over its shard bounds
    (fp32, OpenMP over (request, q-head)).  The reference has no MoE code: the exchange with
    identity experts is a numpy restatement (out_t = sum over t's destination ranks, ascending, of
    that rank's gate-weight sum times x_t), timed with the step.  Returns (tok/s, info)."""
    import bench_multi
    from tests import oracle_lib
    L = oracle_lib.reference()
    if L is None:
        raise RuntimeError("oracle/_ref/libdcpsim_ref.so missing (build with make -C oracle)")
    lens = bench_multi.workload_lens(ws)
    n_all = len(lens)
    cap = (64 * bench_multi.SHORT + (ws - 1) * bench_multi.LONG) // PAGE + 4096
    w = oracle_lib.World(L, "dcpref_", 1, ws, PAGE, cap, "dcp")
    for i, ln in enumerate(lens):
        w.enqueue(i, ln)
    assert len(w.step()["committed"]) == n_all
    pl = [w.placement(i) for i in range(n_all)]
    # bounded sample for host RAM (fp32 K and V: 8 KB per token): every s-th request keeps the mix
    pick = list(range(n_all))
    if token_budget is not None and sum(lens) > token_budget:
        # interleaved order (every s-th request, then the next offset, ...), each taken if it still fits
        s = -(-sum(lens) // token_budget)
        pick, tot = [], 0
        for i in [j for o in range(s) for j in range(o, n_all, s)]:
            if tot + lens[i] <= token_budget:
                pick.append(i)
                tot += lens[i]
        pick.sort()
    sl = np.array([lens[i] for i in pick], np.int64)
    n = len(pick)
    q = np.random.default_rng(0).standard_normal((n, HQ, D), dtype=np.float32)
    kv_off = np.zeros(n, np.int64)
    kv_off[1:] = np.cumsum(sl[:-1] * HKV * D)
    kv_elems = int(sl.sum()) * HKV * D
    k = _tiled(kv_elems, 1)
    v = _tiled(kv_elems, 2)
    bl = [np.cumsum(np.array(pl[i]["split"], np.int64)) for i in pick]   # shard end offsets
    bounds = np.concatenate(bl).astype(np.int64)
    nb = np.array([len(b) for b in bl], np.int32)
    bounds_off = np.zeros(n, np.int64)
    bounds_off[1:] = np.cumsum(nb[:-1])
    out = np.zeros((n, HQ, D), np.float32)
    # MoE: every picked request is one token of its MoE instance; top-k experts and gate weights
    H, E, K = bench_multi.MOE["hidden"], bench_multi.MOE["experts"], bench_multi.MOE["topk"]
    rng = np.random.default_rng(5)
    x = rng.standard_normal((n, H), dtype=np.float32)
    logits = rng.standard_normal((n, E), dtype=np.float32)
    top = np.argsort(-logits, axis=1)[:, :K]
    tv = np.take_along_axis(logits, top, axis=1)
    gw = np.exp(tv - tv.max(axis=1, keepdims=True))
    gw /= gw.sum(axis=1, keepdims=True)
    rank_of = top // (E // ws)
    th = threads or os.cpu_count() or 1
    P = oracle_lib.P
    times = []
    for it in range(warmup + max(steps, 1)):
        t0 = time.perf_counter()
        rc = L.dcpref_batch_decode_attn_f32(n, HQ, HKV, D, 1.0 / math.sqrt(D), P(q), P(k), P(v), P(kv_off),
                                            P(sl), P(bounds), P(bounds_off), P(nb), P(out), th)
        assert rc == 0
        moe_out = np.zeros_like(x)
        for d in range(ws):                      # dispatch -> identity experts -> combine, rank order
            wd = (gw * (rank_of == d)).sum(axis=1)
            rows = np.nonzero(wd)[0]
            moe_out[rows] += wd[rows, None] * x[rows]
        if it >= warmup:
            times.append(time.perf_counter() - t0)
    per_step = float(np.mean(times)) * (sum(lens) / float(sl.sum()))
    full = n == n_all
    what = (f"all {n_all} requests" if full else
            f"{n} of {n_all} requests within a {token_budget}-token budget ({int(sl.sum())} of {sum(lens)} "
            f"KV tokens), scaled by token ratio")
    info = {"kind": "reference", "cores": th,
            "sample": f"{what}: reference Scheduler::step placements (CP histogram "
                      f"{sorted(set(len(p['kv']) for p in pl))}), sharded_attention_merge over each request's "
                      f"shard bounds (fp32) + the MoE exchange with identity experts (numpy; the reference has "
                      f"no MoE code); mean of {len(times)} steps after {warmup} warm-up",
            "same_config": full}
    return n_all / per_step, info


def run_reference(args, ws, rank):
    if rank != 0:
        return
    if ws > 1 and not args.replicas:
        # the N > 1 arm's metric and workload (bench_multi.py)
        import bench_multi
        budget = None if _host_ram_ok(2.5 * (64 * ws * bench_multi.SHORT + (ws - 1) * bench_multi.LONG) * 8192 / 1e9) \
            else 1_000_000
        val, info = cpu_reference_multi(ws, args.steps, args.warmup, token_budget=budget)
        line = {
            "metric": METRIC_MULTI, "value": val, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": len(bench_multi.workload_lens(ws)) / val * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"DCP decode step on {ws} GPUs: per GPU 64 x {bench_multi.SHORT} tokens + "
                                   f"{ws - 1} x {bench_multi.LONG} per node, GQA 32q/8kv d128; then the cfg4 MoE "
                                   f"exchange (identity experts)", "parallelism": "cpu", "l2": "n/a (host)",
                       "requests": len(bench_multi.workload_lens(ws)), "same_config": info["same_config"]},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": info["cores"], "kind": info["kind"],
                             "sample": info["sample"]},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return
    # the whole cfg2 step (1.07M tokens, 8.75 GB of fp32 K/V on the host) when RAM allows
    budget = None if _host_ram_ok(12) else 262_144
    val, info = cpu_reference_sample(args.steps, args.warmup, token_budget=budget)
    line = {
        "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 64.0 / val * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": WORKLOAD, "parallelism": "cpu", "l2": "n/a (host)",
                   "same_config": info["same_config"]},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": info["cores"], "kind": info["kind"],
                         "sample": info["sample"]},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours
def run_ours(args, ws, rank, local):
    import torch
    from paper_2605_21100_b200 import workload
    from paper_2605_21100_b200.attention import DcpContext, DecodeAttention

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    ctx = DcpContext(local)
    # the exact tensors tests/test_attention_gpu.py::test_cfg2_full_size_all_shards checks
    b, pool, q = workload.cfg2_bench_inputs(dev, seed=1234 + rank)
    bt = torch.from_numpy(b.block_table).to(dev)
    cu = torch.from_numpy(b.cu_pages).to(dev)
    sl = torch.from_numpy(b.shard_len).to(dev)
    att = DecodeAttention(ctx, HQ, HKV, D, PAGE, max_shards=64)
    out, lse = att.prepare(q, pool, bt, cu, sl)
    stream = torch.cuda.current_stream(dev)

    for _ in range(max(args.warmup, 3)):
        att.launch(stream)
    torch.cuda.synchronize(dev)
    _barrier(ws)

    # ---- device-timed region: K steps, inputs resident in HBM (> L2: no flush needed)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        evs[0].record(stream)
        for i in range(args.steps):
            att.launch(stream)
            evs[i + 1].record(stream)
        torch.cuda.synchronize(dev)
    ms_total = evs[0].elapsed_time(evs[-1])
    per_step = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)])
    _barrier(ws)
    ms_total = _max_over_ranks(ms_total, ws, dev)
    ms_step = ms_total / args.steps
    value = ws * 64 * args.steps / (ms_total / 1e3)

    # ---- e2e through the C ABI with host buffers: every step copies its own
    # inputs (Q, block table, cu_pages, lengths) from pinned host memory and its
    # result (O, LSE) back, inside the timed region.  Steps are pipelined over
    # three streams with double-buffered device staging: step k+1's H2D overlaps
    # step k's kernel and step k-1's D2H (no step reads another step's data).
    h_q = torch.empty_like(q, device="cpu").pin_memory()
    h_q.copy_(q.cpu())
    h_bt = torch.from_numpy(b.block_table).pin_memory()
    h_cu = torch.from_numpy(b.cu_pages).pin_memory()
    h_sl = torch.from_numpy(b.shard_len).pin_memory()
    h2d = h_q.numel() * 2 + h_bt.numel() * 4 + h_cu.numel() * 4 + h_sl.numel() * 8
    d2h = out.numel() * 4 + lse.numel() * 4
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    sets = []
    for _ in range(2):
        qd, btd, cud, sld = torch.empty_like(q), torch.empty_like(bt), torch.empty_like(cu), torch.empty_like(sl)
        a2 = DecodeAttention(ctx, HQ, HKV, D, PAGE, max_shards=64)
        o2, l2 = a2.prepare(qd, pool, btd, cud, sld)
        sets.append(dict(q=qd, bt=btd, cu=cud, sl=sld, att=a2, out=o2, lse=l2,
                         h_out=torch.empty(o2.shape, dtype=o2.dtype).pin_memory(),
                         h_lse=torch.empty(l2.shape, dtype=l2.dtype).pin_memory(),
                         ev_in=torch.cuda.Event(), ev_k=torch.cuda.Event(), ev_out=torch.cuda.Event()))

    def e2e_steps(n):
        for k in range(n):
            st = sets[k % 2]
            with torch.cuda.stream(s_in):
                s_in.wait_event(st["ev_k"])          # kernel k-2 done reading this staging set
                st["q"].copy_(h_q, non_blocking=True)
                st["bt"].copy_(h_bt, non_blocking=True)
                st["cu"].copy_(h_cu, non_blocking=True)
                st["sl"].copy_(h_sl, non_blocking=True)
                st["ev_in"].record(s_in)
            stream.wait_event(st["ev_in"])
            stream.wait_event(st["ev_out"])          # D2H k-2 done reading this output set
            st["att"].launch(stream)
            st["ev_k"].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(st["ev_k"])
                st["h_out"].copy_(st["out"], non_blocking=True)
                st["h_lse"].copy_(st["lse"], non_blocking=True)
                st["ev_out"].record(s_out)

    e2e_steps(4)
    torch.cuda.synchronize(dev)
    _barrier(ws)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(s_in)
    e2e_steps(args.steps)
    s_in.wait_stream(stream)
    s_in.wait_stream(s_out)
    f1.record(s_in)
    torch.cuda.synchronize(dev)
    e2e_ms = _max_over_ranks(f0.elapsed_time(f1), ws, dev)
    e2e_val = ws * 64 * args.steps / (e2e_ms / 1e3)
    # e2e results must equal the device-resident run
    assert torch.equal(sets[0]["h_out"], out.cpu()) and torch.equal(sets[1]["h_lse"], lse.cpu())

    peak, peak_kind = _peaks()
    alg_bytes = b.algorithmic_bytes()
    achieved = alg_bytes / (ms_step / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- the same step over shuffled frames (a long-running instance after frees), not the
    # fresh-instance LIFO layout above: every page a random 64 KB frame of the pool
    shuffled = None
    if rank == 0 and ws == 1:
        del sets
        b_s, pool_s, q_s = workload.cfg2_bench_inputs(dev, seed=1234 + rank, frame_order="shuffled")
        att_s = DecodeAttention(ctx, HQ, HKV, D, PAGE, max_shards=64)
        att_s.prepare(q_s, pool_s, torch.from_numpy(b_s.block_table).to(dev), torch.from_numpy(b_s.cu_pages).to(dev),
                      torch.from_numpy(b_s.shard_len).to(dev))
        for _ in range(3):
            att_s.launch(stream)
        ns = min(args.steps, 50)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(ns):
            att_s.launch(stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms_s = e0.elapsed_time(e1) / ns
        gbs_s = b_s.algorithmic_bytes() / (ms_s / 1e3) / 1e9
        shuffled = {"frame_order": "shuffled (seeded permutation of 70,925 frames)", "steps": ns, "ms_per_step": ms_s,
                    "tok_s": 64 / (ms_s / 1e3), "achieved_gbs": gbs_s}
        del att_s, pool_s, q_s

    planner = None
    if rank == 0:
        try:
            planner = dict(scenario=PLANNER_SCENARIO, **planner_device(ctx))
        except Exception as e:  # reported, not fatal
            planner = {"scenario": PLANNER_SCENARIO, "error": str(e)}
    mla = None
    if rank == 0 and ws == 1 and not args.no_mla:
        # the cfg5 MLA attention shape on tcgen05 CTA pairs (K10), reported beside K1
        try:
            import bench_mla
            keep = ("workload", "requests", "kv_tokens", "ms_per_step", "decode_tok_s", "achieved_gbs", "hbm_frac",
                    "achieved_tflops", "tensor_frac", "roofline_frac", "peak_kind", "kernel", "gpu_launches_per_step")
            mla = [{k: r[k] for k in keep} for r in bench_mla.run_all(ctx, dev, steps=min(args.steps, 50), warmup=3)]
        except Exception as e:  # reported, not fatal
            mla = {"error": str(e)}
    moe = None
    if rank == 0 and ws == 1 and not args.no_moe:
        # the cfg4 / cfg5 EP exchange (K4 / K5, W = 8 instances emulated on this
        # GPU; peer stores are local), device time per instance of the whole step back to back
        try:
            import bench_moe
            moe = []
            for r in bench_moe.run_all(ctx, dev, steps=min(args.steps, 20), warmup=3):
                moe.append({"workload": r["workload"], "us_per_instance_whole_step": r["whole_step"]["us_per_instance"],
                            "us_p99_per_instance": r["whole_step"]["us_p99_per_instance"],
                            "us_per_instance_event_timed_phases": r["us_per_instance_step"],
                            "cross_instance_bytes_per_step": r["cross_instance_bytes_per_step"],
                            "note": "emulation: one GPU hosts all 8 instances, cross-instance stores are local HBM "
                                    "stores; identity experts; multi-GPU NVLink timing needs an 8-GPU box"})
        except Exception as e:  # reported, not fatal
            moe = {"error": str(e)}
    dcp_p99 = None
    if rank == 0 and ws == 1 and not args.no_dcp:
        # the metric's "P99 step ms": bench_dcp's skewed cfg3-shaped batch (4 instances emulated on
        # this GPU, 3 x 131K + 256 x 2K requests), DCP vs the CP = 1 policies, P99 over 1,000 steps
        try:
            import types
            import bench_dcp
            a = types.SimpleNamespace(instances=4, short_per=64, short_len=2048, long=3, long_len=131073,
                                      capacity=40000, steps=1000, warmup=5, n_sched=8)
            gd = torch.Generator(device=dev).manual_seed(1)
            pools = [torch.randn(a.capacity, 2, 8, 16, 128, generator=gd, device=dev, dtype=torch.bfloat16)
                     for _ in range(a.instances)]
            res = {}
            for pol in ("dcp", "least_batch", "least_cache"):
                r = bench_dcp.run_policy(pol, a, ctx, pools)
                res[pol] = {k: r[k] for k in ("step_ms_p50", "step_ms_p99", "imbalance_pct", "cp_histogram")}
            del pools
            best = min(v["step_ms_p99"] for k, v in res.items() if k != "dcp")
            dcp_p99 = {"workload": "cfg3-shaped skewed batch, 4 instances emulated on one GPU (step = max over "
                                   "instances of the routed K2 + K1 + K3 device time), 1,000 steps",
                       "policies": res, "p99_best_cp1_over_dcp": best / res["dcp"]["step_ms_p99"]}
        except Exception as e:  # reported, not fatal
            dcp_p99 = {"error": str(e)}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            v, info = cpu_reference_sample(2, 1, token_budget=None if _host_ram_ok(12) else 262_144)
            cpu = {"value": v, "unit": UNIT, "cores": info["cores"], "kind": info["kind"],
                   "sample": info["sample"]}
            if planner is not None and "error" not in planner:
                planner.update(planner_cpu_reference())
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOAD, "parallelism": f"replicas x{ws}" if ws > 1 else "single",
                       "l2": "no flush: 4.38 GB KV per step >> 126 MB L2",
                       "kv_tokens": b.total_tokens, "kv_pages": int(b.cu_pages[-1])},
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": "dcp_splitkv_decode_attn via C ABI; per step pinned host Q/block-table/cu/lengths in and O+LSE out, steps pipelined over 3 streams (double-buffered staging)"},
            "gpu_launches": args.steps * _capi_launches(),
            "step_ms_p50": float(np.percentile(per_step, 50)), "step_ms_p99": float(np.percentile(per_step, 99)),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_kind": peak_kind, "kernel": "splitkv_decode_kernel<8,4>",
                         "algorithmic_bytes_per_launch": alg_bytes},
            "shuffled_frames": dict(shuffled, frac=shuffled["achieved_gbs"] / peak) if shuffled else None,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "planner": planner,
            "mla": mla,
            "moe": moe,
            "dcp_p99": dcp_p99,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _capi_launches():
    from paper_2605_21100_b200 import _capi
    return _capi.lib().dcp_attn_launches_per_call()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-mla", action="store_true", help="skip the K10 MLA leg (SURVEY §8f #1)")
    ap.add_argument("--no-moe", action="store_true", help="skip the K4/K5 MoE exchange leg (emulated, 8 instances)")
    ap.add_argument("--no-dcp", action="store_true", help="skip the DCP vs CP=1 P99 leg (emulated, 4 instances)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: N independent cfg2 replicas instead of the multi-GPU DCP step")
    ap.add_argument("--phased", action="store_true",
                    help="N > 1: the routed attention as 4 launches (begin, K2, K1, K3) instead of one fused launch")
    args = ap.parse_args()
    ws, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, ws, rank)
    elif ws > 1 and not args.replicas:
        import bench_multi
        bench_multi.run(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
