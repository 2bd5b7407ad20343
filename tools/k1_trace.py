#!/usr/bin/env python3
"""Per-CTA timeline of one K1 launch (dcp_k1_set_trace): where does a small step's time go?
    python tools/k1_trace.py [--sizes 4x100,16x1000,64x2048]"""
import argparse, ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_21100_b200 import _capi, workload  # noqa: E402
from paper_2605_21100_b200.attention import DcpContext, DecodeAttention  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="4x100,16x1000,64x2048")
ap.add_argument("--fused", action="store_true", help="trace the one-launch routed step (W = 1) instead")
a = ap.parse_args()
dev = torch.device("cuda", 0)
ctx = DcpContext(0)
L = _capi.lib()
for sz in a.sizes.split(","):
    n, ln = map(int, sz.split("x"))
    b = workload.paged_batch([ln] * n, 32, 8, frame_order="shuffled", seed=1)
    pool = torch.randn(b.num_frames, 2, 8, 16, 128, device=dev).to(torch.bfloat16)
    q = torch.randn(n, 32, 128, device=dev).to(torch.bfloat16)
    if a.fused:
        from paper_2605_21100_b200.dcp_step import DcpInstance
        from paper_2605_21100_b200.planner import DevicePlanner
        cap = b.num_frames + 64
        pl = DevicePlanner(ctx, 1, 1, 16, cap, "dcp", None, max_requests=max(64, 2 * n), reserve_pages=8)
        pl.enqueue_many(list(range(n)), [ln] * n)
        pl.step()
        pl.build_routing()
        view = pl.instance_view(0)
        pool = torch.randn(cap, 2, 8, 16, 128, device=dev).to(torch.bfloat16)
        inst = DcpInstance(ctx, 1, 0, 32, 8, cap, kv_pool=pool, n_max=max(512, n), m_max=max(256, n))
        inst.set_peer_local(0, inst)
        inst.commit()
        inst.write_queries(q)

        class _F:
            def launch(self):
                inst.run(view, None, "fused")
        att = _F()
    else:
        att = DecodeAttention(ctx, 32, 8, max_shards=n)
        att.prepare(q, pool, torch.from_numpy(b.block_table).to(dev), torch.from_numpy(b.cu_pages).to(dev),
                    torch.from_numpy(b.shard_len).to(dev))
    for _ in range(5):
        att.launch()
    tr = torch.zeros(ctx.num_sms * 8, dtype=torch.int64, device=dev)
    L.dcp_k1_set_trace(ctypes.c_void_p(tr.data_ptr()))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    att.launch()
    e1.record()
    torch.cuda.synchronize()
    L.dcp_k1_set_trace(None)
    t = tr.cpu().numpy().reshape(-1, 8).astype(np.int64)
    t0 = t[:, 0].min()
    rel = lambda c: np.where(t[:, c] > 0, (t[:, c] - t0) / 1e3, np.nan)  # noqa: E731
    entry, first, seg, tick, merge, ex = (rel(c) for c in range(6))
    print(f"== {sz}: pages {int(b.cu_pages[-1])}, event {e0.elapsed_time(e1)*1e3:.1f} us")
    print(f"   entry us  min {np.nanmin(entry):.2f} median {np.nanmedian(entry):.2f} max {np.nanmax(entry):.2f}")
    print(f"   first stage (after entry) median {np.nanmedian(first - entry):.2f} max {np.nanmax(first - entry):.2f}")
    print(f"   exit us   min {np.nanmin(ex):.2f} median {np.nanmedian(ex):.2f} max {np.nanmax(ex):.2f}")
    print(f"   seg end   median {np.nanmedian(seg):.2f} max {np.nanmax(seg):.2f}; ticket median {np.nanmedian(tick):.2f} "
          f"max {np.nanmax(tick):.2f}; merge (merging CTAs: {int(np.sum(~np.isnan(merge)))}) ticket->done median "
          f"{np.nanmedian(merge - tick):.2f} max {np.nanmax(merge - tick):.2f}")
    o = np.argsort(-np.nan_to_num(ex))[:6]
    for c in o:
        print(f"   slow cta {c:3d} sm {t[c,6]:3d} pages {t[c,7]:3d}: entry {entry[c]:.2f} first {first[c]:.2f} "
              f"seg {seg[c]:.2f} ticket {tick[c]:.2f} merge {merge[c]:.2f} exit {ex[c]:.2f}")
