#!/usr/bin/env python3
"""K1 fixed cost: local K1 over tiny to medium batches, launched 200x back to back from a
prepared argument block (no per-call Python marshalling).  One JSON line per size.

    python tools/probe_k1_small.py [--sizes 1x16,4x100,16x1000,148x16,64x2048]
"""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1x16,4x100,16x1000,148x16,64x2048")
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    import numpy as np, torch
    from paper_2605_21100_b200 import workload
    from paper_2605_21100_b200.attention import DcpContext, DecodeAttention
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    for sz in a.sizes.split(","):
        n, L = map(int, sz.split("x"))
        b = workload.paged_batch([L] * n, 32, 8, frame_order="shuffled", seed=1)
        g = torch.Generator(device=dev).manual_seed(0)
        pool = torch.randn(b.num_frames, 2, 8, 16, 128, generator=g, device=dev).to(torch.bfloat16)
        q = torch.randn(n, 32, 128, generator=g, device=dev).to(torch.bfloat16)
        att = DecodeAttention(ctx, 32, 8, max_shards=n)
        att.prepare(q, pool, torch.from_numpy(b.block_table).to(dev), torch.from_numpy(b.cu_pages).to(dev),
                    torch.from_numpy(b.shard_len).to(dev))
        for _ in range(10):
            att.launch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            att.launch()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / a.iters
        # same launches from a CUDA graph (host enqueue cost removed)
        gr = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(gr, stream=s):
                for _ in range(20):
                    att.launch(s)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        gus = e0.elapsed_time(e1) * 1e3 / 200
        print(json.dumps({"size": sz, "pages": int(b.cu_pages[-1]), "us_eager": us, "us_graph": gus}), flush=True)


if __name__ == "__main__":
    main()
