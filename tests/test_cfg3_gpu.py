"""BASELINE.json configs[2] (cfg3) at full size: the skewed DCP batch.

4 instances (one node), 64 short requests of 2,048 tokens per instance plus 3 long
requests of 131,073 tokens (CP 4 under the default BucketFn, scheduler.cpp:10-33), GQA
32q / 8kv, d = 128, bf16 paged KV, page 16.  One routed step (K2 -> K1 + Res-route -> K3)
over the whole batch; every one of the 259 requests and all 32 heads is checked against
shard_attention<double> + lse_merge over the device page table's per-instance tokens
(bf16 rel-L2 <= 2e-2, LSE <= 1e-5).
"""
import numpy as np
import pytest
import torch

from tests import oracle_lib
from tests.test_dcp_step_gpu import _bits, _oracle_merge
from paper_2605_21100_b200 import workload
from paper_2605_21100_b200._capi import device_to_numpy

pytestmark = pytest.mark.gpu
W, HQ, HKV, D, PAGE, CAP = 4, 32, 8, 128, 16, 16384


def test_cfg3_skewed_batch_full_size():
    from paper_2605_21100_b200.attention import DcpContext
    from paper_2605_21100_b200.dcp_step import DcpInstance, run_local_step
    from paper_2605_21100_b200.planner import DevicePlanner
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    pl = DevicePlanner(ctx, 1, W, PAGE, CAP, "dcp", None, max_requests=512)
    lens = [131073] * 3 + [2048] * (64 * W)
    ids = list(range(len(lens)))
    pl.enqueue_many(ids, lens)
    res = pl.step()
    assert len(res["committed"]) == len(ids)
    longs = [0, 1, 2]
    assert all(len(pl.placement(r)["kv"]) == 4 for r in longs)

    g = torch.Generator(device=dev).manual_seed(3)
    insts = []
    for s in range(W):
        pool = torch.randn(CAP, 2, HKV, PAGE, D, generator=g, device=dev).to(torch.bfloat16)
        insts.append(DcpInstance(ctx, W, s, HQ, HKV, CAP, kv_pool=pool, n_max=512, m_max=256))
    for s in range(W):
        for t in range(W):
            insts[s].set_peer_local(t, insts[t])
        insts[s].commit()
    q = {i: torch.randn(HQ, D, generator=g, device=dev).to(torch.bfloat16) for i in ids}
    out, views = run_local_step(pl, insts, q)
    assert sorted(out) == ids

    check = set(ids)
    port = oracle_lib.port()
    partial = {}
    for s in range(W):
        v = views[s]
        n = v.n_rows
        cu = device_to_numpy(v.cu_pages, n + 1, np.int32)
        nid = device_to_numpy(v.n_ids, n, np.int64)
        sl = device_to_numpy(v.shard_len, n, np.int64)
        bt = device_to_numpy(v.block_table, int(cu[-1]), np.int32)
        fill = device_to_numpy(v.page_fill, int(cu[-1]), np.uint8)
        rows = [j for j in range(n) if int(nid[j]) in check]
        if not rows:
            continue
        cu_s = np.zeros(len(rows) + 1, np.int32)
        for i, j in enumerate(rows):
            cu_s[i + 1] = cu_s[i] + cu[j + 1] - cu[j]
        bt_s = np.concatenate([bt[cu[j]:cu[j + 1]] for j in rows]).astype(np.int32)
        fill_s = np.concatenate([fill[cu[j]:cu[j + 1]] for j in rows]).astype(np.uint8)
        b = workload.PagedBatch(sl[rows].astype(np.int64), cu_s, bt_s, CAP, HQ, HKV)
        qs = torch.stack([q[int(nid[j])] for j in rows])
        o, l = oracle_lib.paged_decode_f64(b, _bits(qs), _bits(insts[s].kv_pool), fill_s)
        for i, j in enumerate(rows):
            partial[(int(nid[j]), s)] = (o[i], l[i])
    worst_o = worst_l = 0.0
    for r in sorted(check):
        p = pl.placement(r)
        for h in range(HQ):
            ro, rl = _oracle_merge(port, [partial[(r, s)][0][h] for s in p["kv"]],
                                   [partial[(r, s)][1][h] for s in p["kv"]], D)
            o, l = out[r][0][h].astype(np.float64), float(out[r][1][h])
            worst_o = max(worst_o, np.linalg.norm(o - ro) / np.linalg.norm(ro))
            worst_l = max(worst_l, abs(l - rl) / max(1.0, abs(rl)))
    print(f"cfg3 all {len(check)} requests x {HQ} heads: worst O rel-L2 {worst_o:.3e}, LSE {worst_l:.3e}")
    assert worst_o <= 2e-2, worst_o
    assert worst_l <= 1e-5, worst_l
    for x in insts:
        x.close()
    pl.close()
