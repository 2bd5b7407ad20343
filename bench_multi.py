"""bench.py at N > 1 GPUs: the real multi-GPU DCP decode step (not replicas).

Launched by bench.py under torchrun, one rank per GPU, one DCP instance per rank.

Workload (BASELINE configs[2] / [3] shapes, weak scaling: fixed work per GPU):
  one node of N instances; per GPU 64 short requests of 2,048 tokens, plus N-1 long
  requests of 131,073 tokens per node (CP min(4, N) under the default BucketFn,
  scheduler.cpp:10-33); GQA 32q / 8kv, d = 128, bf16 paged KV, page 16; then the MoE
  layer of cfg4 (Qwen3-30B-A3B widths: hidden 2,048, 128 experts top-8) over each
  instance's M list with identity experts (the expert GEMMs are library GEMMs, out of
  scope).  Synthetic data.
One step, per rank, with no host synchronisation between ranks:
  begin_step, K2 Q-route puts -> K1 split-KV attention (+ fused Res-route puts) -> K3 LSE
  merge -> begin_step, K4 dispatch -> K5a receive -> identity experts -> K5b combine_put
  -> K5c combine_reduce.
The planner (K6 + K7) runs once as an identical replica on every rank, outside the steps.

value: decode tok/s = requests x steps / max-over-ranks device time.  Per-phase device
times are CUDA events on the step stream (they include cross-rank flag waits); P99 is
over steps of the max-over-ranks step time.  Byte counts are algorithmic.
NCCL baseline (real GPUs only): the same per-step payloads moved with grouped
ncclSend/ncclRecv (torch.distributed.batch_isend_irecv), timed the same way.

DCP_BENCH_ONE_GPU=1 maps every rank to cuda:0 with gloo (a functional check of this
path on one GPU; the ranks then time-slice the device, so the numbers mean nothing).
"""
from __future__ import annotations

import json
import os
import time

import numpy as np

HQ, HKV, D, PAGE = 32, 8, 128, 16
MOE = dict(hidden=2048, experts=128, topk=8, m_max=256)
SHORT, LONG = 2048, 131073


def workload_lens(N):
    return [LONG] * (N - 1) + [SHORT] * (64 * N)


def run(args, ws, rank, local):
    import torch
    import torch.distributed as dist
    from bench import METRIC_MULTI, ClockSampler, UNIT, _peaks
    from paper_2605_21100_b200 import _capi
    from paper_2605_21100_b200._capi import device_to_numpy
    from paper_2605_21100_b200.attention import DcpContext
    from paper_2605_21100_b200.multi import RankStep

    one_gpu = os.environ.get("DCP_BENCH_ONE_GPU") == "1"
    dev_idx = 0 if one_gpu else local
    torch.cuda.set_device(dev_idx)
    dev = torch.device("cuda", dev_idx)
    if one_gpu:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    ctx = DcpContext(dev_idx)
    lens = workload_lens(ws)
    cap = (64 * SHORT + (ws - 1) * LONG) // PAGE + 4096  # any placement fits

    def pool_fn(r, c, h):
        g = torch.Generator(device=dev).manual_seed(77 + r)
        return torch.randn(c, 2, h, PAGE, D, generator=g, device=dev, dtype=torch.bfloat16)

    rs = RankStep(ctx, ws, rank, lens, HQ, HKV, cap, pool_fn, bucket=None, moe=MOE,
                  timeout_ms=60000, n_max=512, m_max=256)
    M = len(rs.m_ids)
    g = torch.Generator(device=dev).manual_seed(5 + rank)
    q = torch.randn(max(M, 1), HQ, D, generator=g, device=dev, dtype=torch.bfloat16)[:M]
    H, E, K = MOE["hidden"], MOE["experts"], MOE["topk"]
    x = torch.randn(max(M, 1), H, generator=g, device=dev, dtype=torch.bfloat16)[:M]
    top = torch.topk(torch.randn(max(M, 1), E, generator=g, device=dev), K, dim=-1)
    idx = top.indices.to(torch.int32)[:M].contiguous()
    wts = torch.softmax(top.values, -1).float()[:M].contiguous()
    stream = torch.cuda.current_stream(dev)

    # ---- algorithmic bytes of this rank
    v = rs.view
    n = v.n_rows
    sl = device_to_numpy(v.shard_len, n, np.int64)
    pages = int(device_to_numpy(v.cu_pages, n + 1, np.int32)[-1])
    k1_bytes = int(sl.sum()) * HKV * D * 2 * 2 + n * (HQ * D * 2 + HQ * D * 4 + HQ * 4) + pages * 4
    pl = rs.planner
    q_out = sum(HQ * D * 2 for r in rs.m_ids for s in pl.placement(r)["kv"] if s != rank)
    res_out = sum(HQ * D * 4 + HQ * 4 for r in rs.n_ids if pl.placement(r)["moe"] != rank)
    per = E // ws
    ranks_of = (idx // per).cpu().numpy() if M else np.zeros((0, K), np.int64)
    disp_out = sum(len(set(rr.tolist()) - {rank}) for rr in ranks_of) * H * 2

    phases = ["route_q", "attention", "merge", "dispatch", "receive", "experts", "combine_put", "combine_reduce"]

    fused = not getattr(args, "phased", False)

    def step(ev):
        ev[0].record(stream)
        rs.inst.write_queries(q, stream) if M else None
        L = _capi.lib()
        import ctypes
        s = ctypes.c_void_p(stream.cuda_stream)
        if fused:  # one launch: fence + Q-route puts + K1 + Res-route + K3 merges (dcp_decode_step_fused)
            ev[1].record(stream)
            rs.inst.run(v, stream, "fused")
            ev[2].record(stream)
        else:
            _capi.check(L.dcp_xchg_begin_step(rs.inst.x, s))
            _capi.check(L.dcp_route_q(rs.inst.x, ctypes.byref(v), s))
            ev[1].record(stream)
            rs.inst.run(v, stream, "attn")
            ev[2].record(stream)
            rs.inst.run(v, stream, "merge")
        ev[3].record(stream)
        m = rs.moe
        m.dispatch(x, idx, wts, m_count_ptr=rs.m_count_ptr, stream=stream, with_receive=fused)
        ev[4].record(stream)
        if not fused:  # fused: K5a runs in K4's last CTA (its time lands in the dispatch phase)
            m.receive_regions(stream)
        ev[5].record(stream)
        m.expert_identity(rs.y_region, stream)  # gate-weighted identity experts (library GEMMs out of scope)
        ev[6].record(stream)
        if fused:  # K5b + K5c in one launch (its time lands in the combine_put phase)
            m.combine_fused(rs.y_region, stream)
            ev[7].record(stream)
        else:
            m.combine_put_regions(rs.y_region, stream)
            ev[7].record(stream)
            m.combine_reduce(stream)
        ev[8].record(stream)

    mk = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(9)]  # noqa: E731
    for _ in range(max(args.warmup, 3)):
        step(mk())
    torch.cuda.synchronize(dev)
    rs.status()
    dist.barrier()
    evs = [mk() for _ in range(args.steps)]
    with ClockSampler(dev_idx) as clk:
        torch.cuda.synchronize(dev)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.steps):
            step(evs[i])
        t1.record(stream)
        torch.cuda.synchronize(dev)
    rs.status()
    total_ms = t0.elapsed_time(t1)
    per_phase = np.array([[e[j].elapsed_time(e[j + 1]) for j in range(8)] for e in evs])  # [steps][8] ms
    per_step = per_phase.sum(axis=1)
    # gather every rank's per-step / per-phase times
    t = torch.tensor(np.concatenate([[total_ms], per_step, per_phase.ravel()]), dtype=torch.float64)
    t = t.to(dev) if not one_gpu else t
    allt = [torch.zeros_like(t) for _ in range(ws)]
    dist.all_gather(allt, t)
    allt = np.stack([a.cpu().numpy() for a in allt])
    tot_max = float(allt[:, 0].max())
    step_max = allt[:, 1:1 + args.steps].max(axis=0)
    ph = allt[:, 1 + args.steps:].reshape(ws, args.steps, 8)
    ph_med = {p: float(np.median(ph[:, :, j].max(axis=0))) * 1e3 for j, p in enumerate(phases)}  # us
    sums = torch.tensor([k1_bytes, q_out, res_out, disp_out, len(rs.m_ids)], dtype=torch.float64)
    sums = sums.to(dev) if not one_gpu else sums
    alls = [torch.zeros_like(sums) for _ in range(ws)]
    dist.all_gather(alls, sums)
    alls = np.stack([a.cpu().numpy() for a in alls])
    n_req = len(lens)
    value = n_req * args.steps / (tot_max / 1e3)
    peak, peak_kind = _peaks()
    k1_us = np.median(ph[:, :, 1], axis=1) * 1e3  # per rank
    k1_gbs = [float(alls[r, 0] / (k1_us[r] * 1e-6) / 1e9) for r in range(ws)]

    nccl = None
    if not one_gpu:
        try:
            nccl = nccl_baseline(ws, rank, dev, alls, args)
        except Exception as e:  # reported, not fatal
            nccl = {"error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC_MULTI, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": tot_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"DCP decode step on {ws} GPUs: per GPU 64 x {SHORT} tokens + {ws - 1} x {LONG} "
                                   f"per node (CP {min(4, ws)}), GQA 32q/8kv d128 bf16 paged; then the cfg4 MoE "
                                   f"exchange (hidden {H}, {E} experts top-{K}, identity experts)",
                       "parallelism": f"dcp{ws} + ep{ws}" + (" (emulated on one GPU)" if one_gpu else ""),
                       "requests": n_req, "l2": "no flush: per-GPU KV >> L2"},
            "step_ms_p50": float(np.percentile(step_max, 50)), "step_ms_p99": float(np.percentile(step_max, 99)),
            "phase_us_median_max_over_ranks": ph_med,
            "k1_hbm_gbs_per_rank": k1_gbs, "k1_hbm_frac_min": min(k1_gbs) / peak, "peak_kind": peak_kind,
            "exchange": {
                "q_route_bytes": float(alls[:, 1].sum()), "res_route_bytes": float(alls[:, 2].sum()),
                "moe_dispatch_bytes": float(alls[:, 3].sum()), "moe_combine_bytes": float(alls[:, 3].sum()),
                "q_route_gbs_per_rank": float(alls[:, 1].mean() / (ph_med["route_q"] * 1e-6) / 1e9),
                "moe_dispatch_gbs_per_rank": float(alls[:, 3].mean() / (ph_med["dispatch"] * 1e-6) / 1e9),
                "moe_combine_gbs_per_rank": float(alls[:, 3].mean() / (ph_med["combine_put"] * 1e-6) / 1e9),
            },
            "nccl_baseline": nccl,
            "attention_launch": "dcp_decode_step_fused (one launch per step)" if fused else "phased (4 launches)",
            "gpu_launches": args.steps * (4 if fused else 9),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    rs.close()
    dist.destroy_process_group()


def nccl_baseline(ws, rank, dev, alls, args):
    """The same per-step exchange volumes through grouped ncclSend / ncclRecv: Q rows out and
    partial rows back (DCP), token rows out and back (MoE).  Each rank sends every peer an
    equal share of its algorithmic bytes (the tables' exact per-peer split differs little at
    these sizes); timed with CUDA events, median over steps, max over ranks."""
    import torch
    import torch.distributed as dist
    res = {}
    for name, col in (("q_route", 1), ("res_route", 2), ("moe_dispatch", 3)):
        nbytes = int(alls[rank, col])
        per_peer = max(16, (nbytes // max(ws - 1, 1)) // 16 * 16)
        send = [torch.empty(per_peer, dtype=torch.uint8, device=dev) for _ in range(ws)]
        recv = [torch.empty(per_peer, dtype=torch.uint8, device=dev) for _ in range(ws)]
        ops = []
        for p in range(ws):
            if p == rank:
                continue
            ops.append(dist.P2POp(dist.isend, send[p], p))
            ops.append(dist.P2POp(dist.irecv, recv[p], p))
        times = []
        for it in range(args.warmup + min(args.steps, 50)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            b.record()
            torch.cuda.synchronize(dev)
            if it >= args.warmup:
                times.append(a.elapsed_time(b) * 1e3)
        t = torch.tensor([float(np.median(times))], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name + "_us"] = float(t.item())
        res[name + "_gbs_per_rank"] = nbytes / (float(t.item()) * 1e-6) / 1e9
    return res
