"""K10 MLA decode-attention bench (the cfg5 DeepSeek-V3 attention shape).

One step = one dcp_mla_decode_attn call (tile scan + the CTA-pair kernel) over a
resident paged bf16 latent cache: 128 heads, 576-wide rows (512 latent + 64 rope),
page 16.  Workloads:
  cfg2-shaped: 64 requests, uniform_int(mt19937_64(0), 1024, 32768) (1.07M tokens,
               1.23 GB of cache per step > L2, so no flush is needed)
  long-mix:    one 524,288-token request + 63 requests uniform_int(mt19937_64(7), 1024, 8192)
Reported per workload: decode tok/s, algorithmic HBM GB/s and tensor TFLOP/s with
their fractions of the measured (or fallback) peaks, and the roofline fraction
= max(bytes / HBM peak, flops / bf16 peak) / measured time.

python bench_mla.py [--steps K] [--warmup W]   (prints one JSON line per workload)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HEADS, DK, DV = 128, 576, 512
PAGE = int(os.environ.get("DCP_MLA_PAGE", "16"))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        # K10 is timed alone over a short run: the burst bf16 figure is its tensor peak
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured (burst bf16)"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def workloads():
    from paper_2605_21100_b200 import workload
    return {
        "cfg2-shaped (64 req, KV 1K-32K)": workload.cfg2_lengths(),
        "long-mix (1 x 512K + 63 x 1K-8K)": [524288] + workload.lengths(7, 63, 1024, 8192),
    }


def alg_bytes(b):
    R = len(b.shard_len)
    return (int(b.shard_len.sum()) * DK * 2 + R * (HEADS * DK * 2 + HEADS * DV * 4 + HEADS * 4)
            + int(b.cu_pages[-1]) * 4)


def alg_flops(b):
    return 2.0 * int(b.shard_len.sum()) * HEADS * (DK + DV)


def inputs(dev, lens):
    """The bench's own batch, cache pool and queries (device, seeded): tests check these."""
    import torch
    from paper_2605_21100_b200 import workload
    b = workload.paged_batch(lens, HEADS, 1, DK, PAGE)
    g = torch.Generator(device=dev).manual_seed(99)
    pool = torch.randn(b.num_frames, PAGE, DK, generator=g, device=dev, dtype=torch.bfloat16)
    q = torch.randn(len(lens), HEADS, DK, generator=g, device=dev, dtype=torch.bfloat16)
    return b, pool, q


def run_workload(ctx, dev, name, lens, steps, warmup):
    import torch
    from paper_2605_21100_b200 import workload
    from paper_2605_21100_b200.attention import MlaDecodeAttention
    b, pool, q = inputs(dev, lens)
    att = MlaDecodeAttention(ctx, PAGE, max_shards=len(lens))
    att.prepare(q, pool, torch.from_numpy(b.block_table).to(dev), torch.from_numpy(b.cu_pages).to(dev),
                torch.from_numpy(b.shard_len).to(dev))
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(warmup, 3)):
        att.launch(stream)
    torch.cuda.synchronize(dev)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    evs[0].record(stream)
    for i in range(steps):
        att.launch(stream)
        evs[i + 1].record(stream)
    torch.cuda.synchronize(dev)
    per = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(steps)])
    ms = float(per.mean())
    hbm, tf, kind = peaks()
    by, fl = alg_bytes(b), alg_flops(b)
    gbs = by / (ms / 1e3) / 1e9
    tfs = fl / (ms / 1e3) / 1e12
    t_roof = max(by / (hbm * 1e9), fl / (tf * 1e12))
    return {
        "workload": name, "requests": len(lens), "kv_tokens": int(b.shard_len.sum()),
        "ms_per_step": ms, "step_ms_p50": float(np.percentile(per, 50)), "step_ms_p99": float(np.percentile(per, 99)),
        "decode_tok_s": len(lens) / (ms / 1e3),
        "achieved_gbs": gbs, "hbm_frac": gbs / hbm, "achieved_tflops": tfs, "tensor_frac": tfs / tf,
        "roofline_frac": t_roof / (ms / 1e3), "peak_kind": kind, "peaks": {"hbm_gbs": hbm, "bf16_tflops": tf},
        "algorithmic_bytes_per_launch": by, "algorithmic_flops_per_launch": fl,
        "kernel": "mla_decode_kernel<16> (tcgen05 cta_group::2) + mla_tile_scan_kernel + mla_merge_kernel",
        "gpu_launches_per_step": 3,
    }


def run_all(ctx, dev, steps=50, warmup=5, only=None):
    res = []
    for name, lens in workloads().items():
        if only and only not in name:
            continue
        res.append(run_workload(ctx, dev, name, lens, steps, warmup))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    import torch
    from paper_2605_21100_b200.attention import DcpContext
    dev = torch.device("cuda", 0)
    ctx = DcpContext(0)
    for r in run_all(ctx, dev, args.steps, args.warmup, args.only):
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
