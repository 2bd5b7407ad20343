#!/usr/bin/env python3
"""Where does a small routed DCP step spend its time?  (the routed
small-step floor.)

One instance (W = 1), 16 requests x 1,000 tokens (or --reqs/--len), GQA 32q/8kv d128 bf16.
Times 200 back-to-back launches of each phase alone and of the whole step with CUDA events
around the loop (so launch gaps count), plus the plain local K1 on the same pages.

    python tools/step_breakdown.py [--reqs 16] [--len 1000] [--world 1]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reqs", type=int, default=16)
    ap.add_argument("--len", type=int, default=1000)
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2605_21100_b200 import _capi
    from paper_2605_21100_b200._capi import device_to_numpy
    from paper_2605_21100_b200.attention import DcpContext, DecodeAttention
    from paper_2605_21100_b200.dcp_step import DcpInstance
    from paper_2605_21100_b200.planner import DevicePlanner

    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    cap = args.reqs * ((args.len + 15) // 16) + 64
    pl = DevicePlanner(ctx, 1, 1, 16, cap, "dcp", None, max_requests=1024, reserve_pages=8)
    g = torch.Generator(device=dev).manual_seed(0)
    pool = torch.randn(cap, 2, 8, 16, 128, generator=g, device=dev).to(torch.bfloat16)
    pl.enqueue_many(list(range(args.reqs)), [args.len] * args.reqs)
    pl.step()
    pl.build_routing()
    view = pl.instance_view(0)
    inst = DcpInstance(ctx, 1, 0, 32, 8, cap, kv_pool=pool, n_max=512, m_max=256)
    inst.set_peer_local(0, inst)
    inst.commit()
    mids = device_to_numpy(view.m_ids, view.m_rows, np.int64)
    q = torch.randn(len(mids), 32, 128, generator=g, device=dev).to(torch.bfloat16)
    inst.write_queries(q)
    L = _capi.lib()
    s = torch.cuda.current_stream(dev)
    sp = __import__("ctypes").c_void_p(s.cuda_stream)
    K = args.iters

    def timed(fn):
        for _ in range(10):
            fn()
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(K):
            fn()
        b.record()
        torch.cuda.synchronize(dev)
        return a.elapsed_time(b) * 1e3 / K

    import ctypes
    out = {"reqs": args.reqs, "len": args.len}
    out["step_us"] = timed(lambda: inst.run(view, None, "all"))
    out["fused_us"] = timed(lambda: inst.run(view, None, "fused"))

    def graphed(phase, n=20):
        gr = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            with torch.cuda.graph(gr, stream=st):
                for _ in range(n):
                    inst.run(view, st, phase)
        torch.cuda.synchronize()
        return timed(gr.replay) / n

    out["step_graph_us"] = graphed("all")
    out["fused_graph_us"] = graphed("fused")
    out["begin_us"] = timed(lambda: L.dcp_xchg_begin_step(inst.x, sp))
    out["k2_us"] = timed(lambda: L.dcp_route_q(inst.x, ctypes.byref(view), sp))
    out["k1_routed_us"] = timed(lambda: L.dcp_decode_attn_routed(ctx.handle, inst.x, ctypes.byref(view),
                                                                   ctypes.byref(inst.args), sp))
    out["k3_us"] = timed(lambda: L.dcp_merge_partials(inst.x, ctypes.byref(view), sp))
    # plain local K1 over the same block table
    att = DecodeAttention(ctx, 32, 8, max_shards=args.reqs)
    bt = torch.from_numpy(device_to_numpy(view.block_table, int(device_to_numpy(view.cu_pages, view.n_rows + 1, np.int32)[-1]), np.int32)).to(dev)
    cu = torch.from_numpy(device_to_numpy(view.cu_pages, view.n_rows + 1, np.int32)).to(dev)
    sl = torch.from_numpy(device_to_numpy(view.shard_len, view.n_rows, np.int64)).to(dev)
    qq = torch.randn(view.n_rows, 32, 128, generator=g, device=dev).to(torch.bfloat16)
    out["k1_local_us"] = timed(lambda: att(qq, pool, bt, cu, sl))
    out["empty_kernel_us"] = timed(lambda: torch.cuda._sleep(0))
    inst.status()
    kv_bytes = args.reqs * args.len * 4096
    out["kv_bytes"] = kv_bytes
    out["kv_time_at_6.5TBs_us"] = kv_bytes / 6.5e12 * 1e6
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
