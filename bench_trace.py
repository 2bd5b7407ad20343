#!/usr/bin/env python3
"""Trace-driven decode serving on the device path: DCP vs CP=1 baselines.

The simengine-equivalent metrics driver of SURVEY §8(f)#3 over real GPU steps
(SPEC.md:432-460 metrics: per-step latency P50/P99, TPOT, SLO attainment,
HoL events, CP histogram, attention reduction potential, KV-load and batch
imbalance, share of active requests at CP > 1; the formulas are in
paper_2605_21100_b200/metrics.py).  Requests arrive from the reference's gen_trace
(ShareGPT-4o short mix + GitHub-Issue long mix, workload.cpp:73-106); every
n_sched iterations the device planner (K6) admits arrivals; every iteration
each active request decodes one token: append_token (K6), routing (K7), the
routed attention step per instance (K2 + K1 + K3), finished requests are
released.  Single-GPU emulation of a W-instance node: each instance's kernels
are timed alone; the iteration's attention latency is the max over
instances, and the simulated clock advances by layers x that latency.

    python bench_trace.py [--instances 8] [--rate 8] [--duration 20] [--long-ratio 0.01]
    python bench_trace.py --sweep-rates 8,16,32,64 --long-ratio 0.05 --slo-ms 20   (P99-TPOT sweep)

Per layer the iteration follows the simengine's critical path:
  QRoute -> Attn -> ResRoute -> Merge (K2 + K1 + K3, per instance)
  -> DS (K4) -> [barrier: DR starts at max_j DS.finish(j)] -> DR (K5a) -> MLP -> CS (K5b)
  -> [barrier] -> CR (K5c)
with every phase but MLP measured on the device for each instance (the MoE exchange of
--moe-hidden / --moe-experts / --moe-topk over each instance's M list), and MLP from the
linear model mu0 + mu_b * B_s of SPEC.md:398 with mu_b derived from the expert FFN's
flops at --mlp-tflops (the expert GEMMs are library GEMMs, out of scope).  --no-moe keeps
the attention-only TPOT of round 1.
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


def run(policy, trace, args, ctx, pools):
    import torch
    from paper_2605_21100_b200 import metrics
    from paper_2605_21100_b200.dcp_step import DcpInstance
    from paper_2605_21100_b200.planner import DevicePlanner
    from paper_2605_21100_b200._capi import device_to_numpy

    W, HQ, HKV = args.instances, 32, 8
    dev = torch.device("cuda:0")
    pl = DevicePlanner(ctx, 1, W, 16, args.capacity, policy, None, hol_strict=True,
                       uniform_degree=args.uniform_degree, max_requests=4096, reserve_pages=64)
    insts = [DcpInstance(ctx, W, s, HQ, HKV, args.capacity, kv_pool=pools[s], n_max=512, m_max=256)
             for s in range(W)]
    for s in range(W):
        for t in range(W):
            insts[s].set_peer_local(t, insts[t])
        insts[s].commit()
    g = torch.Generator(device=dev).manual_seed(11)
    qbank = torch.randn(64, HQ, 128, generator=g, device=dev).to(torch.bfloat16)
    moes = []
    if args.moe:
        from paper_2605_21100_b200.moe import MoeInstance
        Hm, Em, Km = args.moe_hidden, args.moe_experts, args.moe_topk
        moes = [MoeInstance(ctx, W, s, Hm, Km, Em, 256) for s in range(W)]
        for s in range(W):
            for t in range(W):
                moes[s].set_peer_local(t, moes[t])
            moes[s].commit()
        xbank = torch.randn(256, Hm, generator=g, device=dev).to(torch.bfloat16)
        top = torch.topk(torch.randn(256, Em, generator=g, device=dev), Km, dim=-1)
        ibank = top.indices.to(torch.int32).contiguous()
        wbank = torch.softmax(top.values, -1).float().contiguous()
        yreg = [torch.zeros(W, 256, Hm, dtype=torch.bfloat16, device=dev) for _ in range(W)]
        # MLP model: mu0 + mu_b * B_s, mu_b = one token's top-k expert FFN flops
        # (3 GEMMs of hidden x moe_intermediate) at --mlp-tflops
        mu_b_ms = Km * 3 * 2 * Hm * args.moe_intermediate / (args.mlp_tflops * 1e12) * 1e3
    moe_ms, mlp_ms, layer_ms = [], [], []
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t_ms, it = 0.0, 0
    nxt = 0
    queued = set()
    active, remaining, start, out_len = [], {}, {}, {}
    step_ms, tpot, cp_of, hol, sched_ms = [], [], {}, 0, []
    red_attn, kv_imb, b_imb, cp_frac = [], [], [], []
    finished = 0
    while it < args.max_iters:
        if it % args.n_sched == 0:
            new = []
            while nxt < len(trace) and trace[nxt][1] <= t_ms:
                new.append(trace[nxt])
                nxt += 1
            if new:
                pl.enqueue_many([r[0] for r in new], [r[2] for r in new])
                for r in new:
                    queued.add(r[0])
                    out_len[r[0]] = r[3]
            if queued:
                a, b = ev(), ev()
                a.record()
                pl.step_async()
                b.record()
                res = pl.step_result()
                sched_ms.append(a.elapsed_time(b))
                hol += res["hol_events"]
                for rid in res["committed"]:
                    queued.discard(rid)
                    active.append(rid)
                    remaining[rid] = out_len[rid]
                    start[rid] = t_ms
                    cp_of[rid] = len(pl.placement(rid)["kv"])
                for rid in res["unschedulable"]:
                    queued.discard(rid)
        if not active:
            if nxt >= len(trace) and not queued:
                break
            t_ms = max(t_ms, trace[nxt][1]) if nxt < len(trace) else t_ms + 1.0
            it += 1
            continue
        pl.append_many(active)
        ins = pl.instances()
        kv_imb.append(metrics.imbalance_metrics(ins["kv_load"])[0])
        b_imb.append(metrics.imbalance_metrics(ins["moe_batch"])[0])
        cp_frac.append(sum(1 for r in active if cp_of[r] > 1) / len(active))
        pl.build_routing()
        views = [pl.instance_view(s) for s in range(W)]
        for s in range(W):
            v = views[s]
            mids = device_to_numpy(v.m_ids, v.m_rows, np.int64)
            if len(mids):
                insts[s].write_queries(qbank[torch.from_numpy(mids % 64).to(dev)])
        per = [0.0] * W
        marks = []
        gate(ctx)  # host enqueues the whole step behind a device sleep: events time device work only
        for ph in ("q", "attn", "merge"):
            for s in range(W):
                a, b = ev(), ev()
                a.record()
                insts[s].run(views[s], None, ph)
                b.record()
                marks.append((s, a, b))
        mph = {}
        if moes:
            for ph in ("ds", "dr", "cs", "cr"):
                for s in range(W):
                    a, b = ev(), ev()
                    a.record()
                    m = moes[s]
                    if ph == "ds":
                        m.dispatch(xbank, ibank, wbank, m_count_ptr=views[s].m_count_all + 4 * s)
                    elif ph == "dr":
                        m.receive_regions()
                        m.expert_identity(yreg[s])  # stand-in output for CS (the MLP is modelled)
                    elif ph == "cs":
                        m.combine_put_regions(yreg[s])
                    else:
                        m.combine_reduce()
                    b.record()
                    mph[(ph, s)] = (a, b)
        torch.cuda.synchronize(dev)
        for s, a, b in marks:
            per[s] += a.elapsed_time(b)
        attn_lat = max(per)
        lat = attn_lat
        if moes:
            # SPEC.md:422-427 critical path over the measured phases
            t = lambda ph, s: mph[(ph, s)][0].elapsed_time(mph[(ph, s)][1])  # noqa: E731
            bsz = [views[s].m_rows for s in range(W)]
            mlp = [args.mlp_mu0_us / 1e3 + mu_b_ms * bsz[s] for s in range(W)]
            ds_end = [per[s] + t("ds", s) for s in range(W)]
            dr_end = [max(ds_end) + t("dr", s) for s in range(W)]
            cs_end = [dr_end[s] + mlp[s] + t("cs", s) for s in range(W)]
            cr_end = [max(cs_end) + t("cr", s) for s in range(W)]
            lat = max(cr_end)
            moe_ms.append(lat - attn_lat - max(mlp))
            mlp_ms.append(max(mlp))
        step_ms.append(attn_lat)
        layer_ms.append(lat)
        red_attn.append(metrics.imbalance_metrics(per)[1])
        t_ms += args.layers * lat
        done = []
        for rid in active:
            remaining[rid] -= 1
            if remaining[rid] <= 0:
                done.append(rid)
        for rid in done:
            pl.finish(rid)
            active.remove(rid)
            tpot.append((t_ms - start[rid]) / out_len[rid])
            finished += 1
        it += 1
    for x in insts + moes:
        x.close()
    pl.close()
    st, tp = np.array(step_ms), np.array(tpot) if tpot else np.array([0.0])
    ks = list(cp_of.values())
    return {
        "policy": policy if policy != "uniform" else f"uniform{args.uniform_degree}",
        "iterations": len(step_ms), "finished": finished, "admitted": len(cp_of),
        "step_ms_p50": float(np.percentile(st, 50)), "step_ms_p99": float(np.percentile(st, 99)),
        "step_ms_max": float(st.max()),
        "tpot_ms_mean": float(tp.mean()), "tpot_ms_p99": float(np.percentile(tp, 99)),
        "slo_attainment": metrics.slo_attainment(tpot, args.slo_ms),
        "hol_events": hol, "cp_histogram": {str(k): ks.count(k) for k in sorted(set(ks))},
        "planner_step_ms_mean": float(np.mean(sched_ms)) if sched_ms else None,
        # SPEC.md:432-439 formulas over the per-iteration per-instance values (AC5, AC6, AC8)
        "attn_reduction_potential_pct_mean": float(np.mean(red_attn)) if red_attn else 0.0,
        "kv_load_imbalance_pct_mean": float(np.mean(kv_imb)) if kv_imb else 0.0,
        "batch_imbalance_pct_mean": float(np.mean(b_imb)) if b_imb else 0.0,
        "cp_gt1_active_frac_max": float(max(cp_frac)) if cp_frac else 0.0,
        "cp_gt1_active_frac_mean": float(np.mean(cp_frac)) if cp_frac else 0.0,
        "sim_time_s": t_ms / 1e3,
        "layer_model": ("attention + MoE exchange measured, MLP modelled (SPEC.md:422-427 critical path)"
                        if moes else "attention only"),
        "layer_ms_p50": float(np.percentile(layer_ms, 50)) if layer_ms else None,
        "layer_ms_p99": float(np.percentile(layer_ms, 99)) if layer_ms else None,
        "moe_exchange_ms_per_layer_p50": float(np.percentile(moe_ms, 50)) if moe_ms else None,
        "mlp_model_ms_per_layer_p50": float(np.percentile(mlp_ms, 50)) if mlp_ms else None,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", type=int, default=8)
    ap.add_argument("--capacity", type=int, default=64000)
    ap.add_argument("--rate", type=float, default=8.0)
    ap.add_argument("--duration", type=float, default=20.0)
    ap.add_argument("--long-ratio", type=float, default=0.01)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--out-min", type=int, default=32)
    ap.add_argument("--out-max", type=int, default=128)
    ap.add_argument("--layers", type=int, default=48, help="attention layers per decode iteration")
    ap.add_argument("--slo-ms", type=float, default=50.0)
    ap.add_argument("--n-sched", type=int, default=4)
    ap.add_argument("--max-iters", type=int, default=4000)
    ap.add_argument("--uniform-degree", type=int, default=8)
    ap.add_argument("--policies", default="dcp,least_batch,least_cache,uniform")
    ap.add_argument("--no-moe", dest="moe", action="store_false",
                    help="attention-only TPOT (no DS/DR/MLP/CS/CR phases)")
    ap.add_argument("--moe-hidden", type=int, default=2048, help="cfg4 (Qwen3-30B-A3B) hidden size")
    ap.add_argument("--moe-experts", type=int, default=128)
    ap.add_argument("--moe-topk", type=int, default=8)
    ap.add_argument("--moe-intermediate", type=int, default=768)
    ap.add_argument("--mlp-tflops", type=float, default=800.0,
                    help="effective bf16 TFLOP/s of the expert GEMMs in the MLP model")
    ap.add_argument("--mlp-mu0-us", type=float, default=10.0, help="fixed MLP cost per layer (mu0)")
    ap.add_argument("--trace-csv", default="",
                    help="replay this trace file (the reference's id,arrival_ms,seq_len,output_len format, "
                         "workload.cpp:108-137) instead of generating one")
    ap.add_argument("--write-trace", default="",
                    help="write the generated trace to this CSV file (write_trace_csv format) before replaying it")
    ap.add_argument("--sweep-rates", default="",
                    help="comma-separated ascending rates: P99-TPOT sweep + max sustainable rate (SPEC.md:449-455)")
    args = ap.parse_args()
    import torch
    from paper_2605_21100_b200 import metrics, workload
    from paper_2605_21100_b200.attention import DcpContext
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(1)
    pools = [torch.randn(args.capacity, 2, 8, 16, 128, generator=g, device=dev, dtype=torch.bfloat16)
             for _ in range(args.instances)]
    setup = (f"{args.instances} instances (single-GPU emulation), GQA 32q/8kv d128 bf16, "
             f"{args.layers} layers/iteration, SLO {args.slo_ms} ms TPOT "
             + (f"(attention + MoE exchange hidden {args.moe_hidden} / {args.moe_experts} experts top-{args.moe_topk} "
                f"measured, MLP modelled at {args.mlp_tflops} TFLOP/s)" if args.moe else "(attention layers only)"))
    rates = [float(x) for x in args.sweep_rates.split(",") if x] or [args.rate]
    by_policy = {}
    for rate in rates:
        if args.trace_csv:
            with open(args.trace_csv) as f:
                trace = workload.load_trace_csv(f.read())
        else:
            trace = workload.gen_trace(args.seed, args.long_ratio, rate, args.duration, poisson=True,
                                       output_len=(args.out_min, args.out_max))
            if args.write_trace:
                with open(args.write_trace, "w") as f:
                    f.write(workload.write_trace_csv(trace))
                # replay exactly what the file holds (arrivals rounded to the file's 3 decimals)
                trace = workload.load_trace_csv(workload.write_trace_csv(trace))
        longs = sum(1 for r in trace if r[2] >= 100000)
        print(json.dumps({"trace": {"requests": len(trace), "long": longs, "rate_per_s": rate,
                                    "duration_s": args.duration, "long_ratio": args.long_ratio,
                                    "max_len": max(r[2] for r in trace)}, "setup": setup}), flush=True)
        results = []
        for pol in args.policies.split(","):
            r = run(pol, trace, args, ctx, pools)
            r["rate_per_s"] = rate
            results.append(r)
            by_policy.setdefault(r["policy"], []).append(r)
            print(json.dumps(r), flush=True)
        dcp = next((r for r in results if r["policy"] == "dcp"), None)
        base = [r for r in results if r["policy"] != "dcp"]
        if dcp and base:
            best = min(base, key=lambda r: r["step_ms_p99"])
            print(json.dumps({"rate_per_s": rate, "p99_step_dcp_vs_best_baseline": best["step_ms_p99"] / dcp["step_ms_p99"],
                              "best_baseline": best["policy"]}), flush=True)
    if len(rates) > 1:
        summary = {"sweep": "P99 TPOT (ms) per rate and max sustainable rate at SLO "
                            f"{args.slo_ms} ms / 99% (SPEC.md:449-455, monotone truncation)", "rates": rates}
        for pol, rs in by_policy.items():
            att = {r["rate_per_s"]: r["slo_attainment"] for r in rs}
            best, _ = metrics.slo_sweep(att.__getitem__, rates)
            summary[pol] = {"tpot_ms_p99": [r["tpot_ms_p99"] for r in rs],
                            "step_ms_p99": [r["step_ms_p99"] for r in rs],
                            "slo_attainment": [r["slo_attainment"] for r in rs],
                            "hol_events": [r["hol_events"] for r in rs],
                            "attn_reduction_potential_pct": [round(r["attn_reduction_potential_pct_mean"], 1) for r in rs],
                            "kv_load_imbalance_pct": [round(r["kv_load_imbalance_pct_mean"], 1) for r in rs],
                            "batch_imbalance_pct": [round(r["batch_imbalance_pct_mean"], 1) for r in rs],
                            "max_sustainable_rate": best}
        print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
