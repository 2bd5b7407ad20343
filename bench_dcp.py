#!/usr/bin/env python3
"""DCP vs CP=1 (LeastBatch / LeastCache) decode-attention step latency on a
long/short skewed batch (BASELINE configs[2]), on the same kernels.

Single-GPU emulation of a W-instance node (the mode this round's 1-GPU budget
allows): every instance's routed step — Q-route puts (K2), split-KV attention
with fused Res-route puts (K1), LSE merge (K3) — runs on the one B200 with its
own KV pool, page table view and exchange pools; each instance's kernels are
timed alone with CUDA events, and the step latency is the max over instances
(the critical path if each instance had its own GPU; the NVLink hops are local
stores here).  Every step decodes one token per request (append_token on the
device planner) and re-derives the routing (K7); the planner's own step (K6)
and routing build are timed separately.

    python bench_dcp.py [--instances 4] [--steps 300] [--long 3] [--long-len 131072]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def gate(ctx, us=3000):
    import ctypes
    import torch
    from paper_2605_21100_b200 import _capi
    s = torch.cuda.current_stream(ctx.device).cuda_stream
    _capi.check(_capi.lib().dcp_device_sleep(ctx.handle, us, ctypes.c_void_p(s)))


def run_policy(policy, args, ctx, pools):
    import torch
    from paper_2605_21100_b200.dcp_step import DcpInstance
    from paper_2605_21100_b200.planner import DevicePlanner
    from paper_2605_21100_b200._capi import device_to_numpy

    W, HQ, HKV = args.instances, 32, 8
    dev = torch.device("cuda:0")
    pl = DevicePlanner(ctx, 1, W, 16, args.capacity, policy, None, max_requests=2048, reserve_pages=64)
    # skewed batch: `short_per` 2K requests per instance + `long` long requests, interleaved
    n_short = args.short_per * W
    lens, ids = [], []
    pos_long = set(np.linspace(0, n_short, args.long + 2, dtype=int)[1:-1].tolist())
    rid = 0
    for i in range(n_short + args.long):
        is_long = i in pos_long and sum(1 for L in lens if L == args.long_len) < args.long
        lens.append(args.long_len if is_long else args.short_len)
        ids.append(rid)
        rid += 1
    pl.enqueue_many(ids, lens)
    r = pl.step()
    active = r["committed"]
    insts = [DcpInstance(ctx, W, s, HQ, HKV, args.capacity, kv_pool=pools[s], n_max=512, m_max=512)
             for s in range(W)]
    for s in range(W):
        for t in range(W):
            insts[s].set_peer_local(t, insts[t])
        insts[s].commit()
    g = torch.Generator(device=dev).manual_seed(3)
    q_all = torch.randn(len(ids), HQ, 128, generator=g, device=dev).to(torch.bfloat16)
    import torch.cuda as tc
    ev = lambda: tc.Event(enable_timing=True)  # noqa: E731
    step_ms, inst_ms_all, plan_ms, route_ms = [], [], [], []
    kv_tokens_max, kv_tokens_mean = [], []
    stream = torch.cuda.current_stream(dev)
    for step in range(args.warmup + args.steps):
        # decode growth + (every n_sched steps) a planner round: timed on device
        e0, e1, e2 = ev(), ev(), ev()
        e0.record(stream)
        pl.append_many(active)
        if step % args.n_sched == 0:
            pl.step_async()
        e1.record(stream)
        pl.build_routing()
        e2.record(stream)
        views = [pl.instance_view(s) for s in range(W)]
        for s in range(W):
            v = views[s]
            mids = device_to_numpy(v.m_ids, v.m_rows, np.int64)
            if len(mids):
                insts[s].write_queries(q_all[torch.from_numpy(mids).to(dev)])
        t_q, t_a, t_m = [], [], []
        gate(ctx)  # host enqueues the whole step behind a device sleep: events time device work only
        for s in range(W):
            a, b = ev(), ev()
            a.record(stream)
            insts[s].run(views[s], None, "q")
            b.record(stream)
            t_q.append((a, b))
        for s in range(W):
            a, b = ev(), ev()
            a.record(stream)
            insts[s].run(views[s], None, "attn")
            b.record(stream)
            t_a.append((a, b))
        for s in range(W):
            a, b = ev(), ev()
            a.record(stream)
            insts[s].run(views[s], None, "merge")
            b.record(stream)
            t_m.append((a, b))
        torch.cuda.synchronize(dev)
        if step % args.n_sched == 0:
            pl.step_result()
        if step < args.warmup:
            continue
        per = [t_q[s][0].elapsed_time(t_q[s][1]) + t_a[s][0].elapsed_time(t_a[s][1]) +
               t_m[s][0].elapsed_time(t_m[s][1]) for s in range(W)]
        inst_ms_all.append(per)
        step_ms.append(max(per))
        plan_ms.append(e0.elapsed_time(e1))
        route_ms.append(e1.elapsed_time(e2))
        kv = pl.instances()["kv_load"] if step == args.warmup or step == args.warmup + args.steps - 1 else None
        if kv:
            kv_tokens_max.append(max(kv))
            kv_tokens_mean.append(sum(kv) / len(kv))
    ks = [len(pl.placement(i)["kv"]) for i in active]
    st = np.array(step_ms)
    res = {
        "policy": policy, "instances": W, "requests": len(active), "steps": args.steps,
        "step_ms_p50": float(np.percentile(st, 50)), "step_ms_p99": float(np.percentile(st, 99)),
        "step_ms_mean": float(st.mean()),
        "decode_tok_s": len(active) / (st.mean() / 1e3),
        "instance_ms_mean": [float(x) for x in np.mean(np.array(inst_ms_all), axis=0)],
        "imbalance_pct": float((np.max(np.mean(inst_ms_all, axis=0)) / np.mean(inst_ms_all) - 1) * 100),
        "cp_histogram": {str(k): ks.count(k) for k in sorted(set(ks))},
        "kv_load_max_over_mean": [float(a / b) for a, b in zip(kv_tokens_max, kv_tokens_mean)],
        "planner_append_step_ms_mean": float(np.mean(plan_ms)),
        "routing_build_ms_mean": float(np.mean(route_ms)),
    }
    for x in insts:
        x.close()
    pl.close()
    return res


def run_multi(args):
    """One instance per rank (torchrun): the routed step with real peer stores
    over NVLink between GPUs.  The planner runs as an identical replica on
    every rank (checked by digest); ranks step in lock-step (host barrier
    between steps, outside the timed region); step latency = max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2605_21100_b200 import multi
    from paper_2605_21100_b200.attention import DcpContext
    from paper_2605_21100_b200.dcp_step import DcpInstance
    from paper_2605_21100_b200.planner import DevicePlanner
    from paper_2605_21100_b200._capi import device_to_numpy

    rank, ws, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ctx = DcpContext(local)
    results = []
    for policy in args.policies.split(","):
        pl = DevicePlanner(ctx, 1, ws, 16, args.capacity, policy, None, max_requests=2048, reserve_pages=64)
        n_short = args.short_per * ws
        pos_long = set(np.linspace(0, n_short, args.long + 2, dtype=int)[1:-1].tolist())
        lens = [args.long_len if i in pos_long else args.short_len for i in range(n_short + args.long)]
        ids = list(range(len(lens)))
        pl.enqueue_many(ids, lens)
        active = pl.step()["committed"]
        g = torch.Generator(device=dev).manual_seed(1 + rank)
        pool = torch.randn(args.capacity, 2, 8, 16, 128, generator=g, device=dev, dtype=torch.bfloat16)
        inst = DcpInstance(ctx, ws, rank, 32, 8, args.capacity, kv_pool=pool, n_max=512, m_max=512)
        multi.connect_peers(inst, multi.exchange_handles(inst.ipc_handle()))
        pl.build_routing()
        multi.check_replicas(pl.routing_csv())
        q_all = torch.randn(len(ids), 32, 128, generator=torch.Generator(device=dev).manual_seed(3), device=dev
                            ).to(torch.bfloat16)
        steps = []
        for step in range(args.warmup + args.steps):
            pl.append_many(active)
            pl.build_routing()
            v = pl.instance_view(rank)
            mids = device_to_numpy(v.m_ids, v.m_rows, np.int64)
            if len(mids):
                inst.write_queries(q_all[torch.from_numpy(mids).to(dev)])
            torch.cuda.synchronize(dev)
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            inst.run(v)
            b.record()
            torch.cuda.synchronize(dev)
            if step >= args.warmup:
                steps.append(multi.max_over_ranks(a.elapsed_time(b), dev))
        st = np.array(steps)
        results.append({"policy": policy, "ranks": ws, "requests": len(active),
                        "step_ms_p50": float(np.percentile(st, 50)), "step_ms_p99": float(np.percentile(st, 99)),
                        "step_ms_mean": float(st.mean()), "decode_tok_s": len(active) / (st.mean() / 1e3)})
        dist.barrier()
        inst.close()
        pl.close()
    if rank == 0:
        for r in results:
            print(json.dumps(r), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--multi", action="store_true", help="torchrun: one instance per GPU, real NVLink exchange")
    ap.add_argument("--instances", type=int, default=4)
    ap.add_argument("--short-per", type=int, default=64)
    ap.add_argument("--short-len", type=int, default=2048)
    ap.add_argument("--long", type=int, default=3)
    ap.add_argument("--long-len", type=int, default=131073)
    ap.add_argument("--capacity", type=int, default=40000)
    ap.add_argument("--steps", type=int, default=1000)  # P99 over >= 1,000 steps
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--n-sched", type=int, default=8)
    ap.add_argument("--policies", default="dcp,least_batch,least_cache")
    args = ap.parse_args()
    if args.multi:
        return run_multi(args)
    import torch
    from paper_2605_21100_b200.attention import DcpContext
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(1)
    pools = [torch.randn(args.capacity, 2, 8, 16, 128, generator=g, device=dev, dtype=torch.bfloat16)
             for _ in range(args.instances)]
    out = {"workload": (f"cfg3-shaped single-GPU emulation: {args.instances} instances x {args.short_per} requests "
                        f"@{args.short_len} + {args.long} @{args.long_len}, GQA 32q/8kv d128 bf16 page 16; "
                        f"step latency = max over instances of (K2+K1+K3) device time"),
           "results": []}
    for pol in args.policies.split(","):
        r = run_policy(pol, args, ctx, pools)
        out["results"].append(r)
        print(json.dumps(r), flush=True)
    dcp = next((r for r in out["results"] if r["policy"] == "dcp"), None)
    base = [r for r in out["results"] if r["policy"] != "dcp"]
    if dcp and base:
        best = min(base, key=lambda r: r["step_ms_p99"])
        out["p99_dcp_vs_best_cp1"] = best["step_ms_p99"] / dcp["step_ms_p99"]
    print(json.dumps({k: v for k, v in out.items() if k != "results"}), flush=True)


if __name__ == "__main__":
    main()
