"""Run one K10 call with the pair-0 timeline trace on and print per-tile intervals (ns).
    python tools/mla_trace.py [--page 16] [--dbg 0]"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_21100_b200 import _capi, workload  # noqa: E402
from paper_2605_21100_b200.attention import DcpContext, MlaDecodeAttention  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--page", type=int, default=16)
ap.add_argument("--dbg", type=int, default=0)
args = ap.parse_args()
dev = torch.device("cuda", 0)
ctx = DcpContext(0)
lens = workload.cfg2_lengths()
b = workload.paged_batch(lens, 128, 1, 576, args.page)
pool = torch.randn(b.num_frames, args.page, 576, device=dev, dtype=torch.bfloat16)
q = torch.randn(len(lens), 128, 576, device=dev, dtype=torch.bfloat16)
att = MlaDecodeAttention(ctx, args.page, max_shards=len(lens))
att.prepare(q, pool, torch.from_numpy(b.block_table).to(dev), torch.from_numpy(b.cu_pages).to(dev),
            torch.from_numpy(b.shard_len).to(dev))
for _ in range(3):
    att.launch()
tr = torch.zeros(2048 + 3 * 256, dtype=torch.int64, device=dev)
_capi.lib().dcp_mla_set_trace(ctypes.c_void_p(tr.data_ptr()))
att.launch()
torch.cuda.synchronize()
_capi.lib().dcp_mla_set_trace(None)
allt = tr.cpu().numpy()
t = allt[:2048].reshape(256, 8).copy()
pt = allt[2048:].reshape(256, 3)
npair = int((pt[:, 1] > 0).sum())
pt = pt[:npair]
st0 = pt[:, 0].min()
ends = (pt[:, 1] - st0) / 1e3
starts = (pt[:, 0] - st0) / 1e3
print(f"pairs {npair}: start us min/max {starts.min():.1f}/{starts.max():.1f}; end us min/median/max "
      f"{ends.min():.1f}/{np.median(ends):.1f}/{ends.max():.1f}")
order = np.argsort(ends)
print("slowest pairs (pair, sm, end us):", [(int(i), int(pt[i, 2]), round(float(ends[i]), 1)) for i in order[-8:]])
print("fastest pairs (pair, sm, end us):", [(int(i), int(pt[i, 2]), round(float(ends[i]), 1)) for i in order[:8]])
for row, nm in ((252, "QK-A"), (253, "QK-B"), (254, "PV-0"), (255, "PV-1")):
    print(f"{nm} MMA warp: total ns", t[row, 0], "waiting on full ring ns", t[row, 1], "waits", t[row, 2], "ready", t[row, 3])
t[252:] = 0
n = int((t[:, 0] > 0).sum())
t0 = t[0, 0]
t = t[:n].astype(np.int64) - t0
print("tile  qk_start qk_issued  pfull(g) pv_issued | S_ready P_pub max_done P_free  (CTA0 softmax; ns from tile 0)")
for g in range(n):
    print(f"{g:4d} " + " ".join(f"{x:8d}" for x in t[g]))
d = np.diff(t[:, 0])
print("per-tile period (ns): median", np.median(d), "mean", d.mean())
sm = t[:, 5] - t[:, 4]
print("softmax CTA0 S-ready -> P-published: median", np.median(sm))
print("  S-ready -> max done: median", np.median(t[:, 6] - t[:, 4]), " max done -> P buffer free:", np.median(t[:, 7] - t[:, 6]),
      " P free -> P published:", np.median(t[:, 5] - t[:, 7]))
print("  softmax idle (S-ready(g) - P-pub(g-1)): median", np.median(t[1:, 4] - t[:-1, 5]))
print("S-ready(g) after qk_issued(g): median", np.median(t[:, 4] - t[:, 1]))
print("MMA P(g) wait return after P-published(g) (max of CTAs):", np.median(t[:-1, 2] - np.maximum(t[:-1, 5], t[:-1, 7])))
