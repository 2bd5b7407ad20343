"""AOT step-graph memory (the paper's Table 2).

Creates one instance's exchange pools and its step graphs (dcp_step_graph_create: one
executable graph per M-bucket of ShapeSpace::default_space(), shared by the buckets that
differ only in N) and reports the device memory they take (cudaMemGetInfo deltas), next to
the reference's own estimate for the same shape space (graph_memory_footprint,
routing.cpp:115-127, computed by the oracle port with the reference's default model dims).
The paper's figure (48 graphs, 5.32 GiB per GPU) covers whole-model graphs, so only the
graph counts are directly comparable; the attention-step bytes are reported as measured.
Also timed: the same small routed step replayed from its graph vs launched eagerly.

python bench_graph.py    (one JSON line)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2605_21100_b200.attention import DcpContext
    from paper_2605_21100_b200.dcp_step import DcpInstance, StepGraph
    from paper_2605_21100_b200.planner import DevicePlanner
    from tests import oracle_lib
    from paper_2605_21100_b200._capi import device_to_numpy
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")

    def used():
        torch.cuda.synchronize(dev)
        f, t = torch.cuda.mem_get_info(dev)
        return t - f

    cap = 4096
    pl = DevicePlanner(ctx, 1, 1, 16, cap, "dcp", None, max_requests=1024, reserve_pages=8)
    pool = torch.zeros(cap, 2, 8, 16, 128, dtype=torch.bfloat16, device=dev)
    pl.enqueue_many(list(range(16)), [1000] * 16)
    pl.step()
    pl.build_routing()
    view = pl.instance_view(0)
    u0 = used()
    inst = DcpInstance(ctx, 1, 0, 32, 8, cap, kv_pool=pool, n_max=512, m_max=256)
    inst.set_peer_local(0, inst)
    inst.commit()
    u1 = used()
    sg = StepGraph(inst, view)
    u2 = used()
    L = oracle_lib.port()
    fp = np.zeros(2, np.int64)
    n_graphs = np.zeros(1, np.int64)
    # reference defaults: Hn 128, Hs 64, D 7168, MaxBlk 1024 (routing.hpp:64-70), W = 1 and 8
    ref = {}
    for W in (1, 8):
        rc = L.dcpora_graph_footprint(W, 128, 64, 7168, 1024, 2, 4, oracle_lib.P(n_graphs), oracle_lib.P(fp))
        ref[f"W{W}"] = {"graphs": int(n_graphs[0]), "bytes": int(fp[0]), "rc": int(rc)}
    # replay vs eager: the same routed step (16 requests x 1,000 tokens, W = 1), K launches each,
    # timed with CUDA events around the whole loop (host launch cost included)
    mids = device_to_numpy(view.m_ids, view.m_rows, np.int64)
    g = torch.Generator(device=dev).manual_seed(0)
    inst.write_queries(torch.randn(len(mids), 32, 128, generator=g, device=dev).to(torch.bfloat16))
    K = 200

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

    eager_us = timed(lambda: inst.run(view, None, "all"))
    graph_us = timed(lambda: sg.launch(view.m_rows, view.n_rows))
    line = {
        "metric": "AOT step-graph memory per GPU (routed attention step, 32q/8kv d128, n_max 512, m_max 256)",
        "step_us_eager": eager_us, "step_us_graph": graph_us,
        "step_note": "16 requests x 1,000 tokens on one instance; per-step time over 200 back-to-back steps",
        "buckets": sg.buckets, "executable_graphs": sg.graphs,
        "exchange_pool_bytes": int(u1 - u0), "graph_bytes": int(u2 - u1),
        "reference_graph_memory_footprint": ref,
        "paper_table2": {"graphs": 48, "GiB_per_gpu": 5.32, "scope": "whole-model decode graphs"},
    }
    print(json.dumps(line), flush=True)
    sg.close()


if __name__ == "__main__":
    main()
