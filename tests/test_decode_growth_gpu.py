"""Decode growth and the largest shapes.

* K8 kv_append: after append_token, each request's new K/V lands in the frame
  and slot append_token chose (page_table.cpp:86-121), including fallback
  pages on another instance.
* A 524,288-token request (cfg5 length) at CP 8 over 8 instances (default
  BucketFn, scheduler.cpp:28-33) through the routed step, checked against the
  oracle; plus a decode step with the new token appended by K8.
"""
import numpy as np
import pytest
import torch

from tests import oracle_lib
from tests.test_dcp_step_gpu import _bits, _oracle_merge
from paper_2605_21100_b200 import workload
from paper_2605_21100_b200._capi import device_to_numpy

pytestmark = pytest.mark.gpu
I64MAX = 2**63 - 1


def _ctx():
    from paper_2605_21100_b200.attention import DcpContext
    return DcpContext(0)


def test_kv_append_writes_chosen_slot():
    from paper_2605_21100_b200.planner import DevicePlanner
    ctx = _ctx()
    dev = torch.device("cuda:0")
    W, cap = 4, 64
    pl = DevicePlanner(ctx, 1, W, 16, cap, "dcp", [[40, 1], [160, 2], [I64MAX, 4]], max_requests=64)
    rng = np.random.default_rng(2)
    ids = list(range(24))
    pl.enqueue_many(ids, rng.integers(1, 300, size=24).tolist())
    active = pl.step()["committed"]
    pools = [torch.zeros(cap, 2, 8, 16, 128, dtype=torch.bfloat16, device=dev) for _ in range(W)]
    g = torch.Generator(device=dev).manual_seed(0)
    for rnd in range(20):                      # enough growth to cross pages and hit fallbacks
        got_inst = dict(zip(active, pl.append_many(active).tolist()))
        pl.build_routing()
        pt = [list(map(int, l.split(","))) for l in pl.page_table_csv().strip().split("\n")[1:]]
        last = {}
        for r, p, i, f in pt:
            last[r] = (i, f)
        fills = {}
        for s in range(W):
            v = pl.instance_view(s)
            cu = device_to_numpy(v.cu_pages, v.n_rows + 1, np.int32)
            fl = device_to_numpy(v.page_fill, int(cu[-1]), np.uint8)
            for row, r in enumerate(device_to_numpy(v.n_ids, v.n_rows, np.int64)):
                if last[int(r)][0] == s:
                    fills[int(r)] = int(fl[cu[row + 1] - 1])
        news = {}
        for s in range(W):
            v = pl.instance_view(s)
            mids = device_to_numpy(v.m_ids, v.m_rows, np.int64)
            kv = torch.randn(len(mids), 2, 8, 128, generator=g, device=dev).to(torch.bfloat16)
            if len(mids):
                pl.kv_append(s, kv, pools)
            for j, r in enumerate(mids):
                news[int(r)] = kv[j]
        torch.cuda.synchronize()
        for r in active:
            if got_inst[r] < 0:                # growth stall: nothing written
                continue
            inst, frame = last[r]
            slot = fills[r] - 1
            got = pools[inst][frame, :, :, slot, :]
            assert torch.equal(got, news[r]), (rnd, r)


def test_512k_request_cp8_routed_step():
    from paper_2605_21100_b200.dcp_step import DcpInstance, run_local_step
    from paper_2605_21100_b200.planner import DevicePlanner
    ctx = _ctx()
    dev = torch.device("cuda:0")
    W, cap, hq, hkv = 8, 6000, 32, 8
    pl = DevicePlanner(ctx, 1, W, 16, cap, "dcp", None, max_requests=64, reserve_pages=16)
    lens = [524288, 3000, 17, 40000, 1]
    pl.enqueue_many(list(range(len(lens))), lens)
    res = pl.step()
    assert res["committed"] == list(range(len(lens)))
    assert len(pl.placement(0)["kv"]) == 8 and sum(pl.placement(0)["split"]) == 524288
    g = torch.Generator(device=dev).manual_seed(5)
    insts = []
    for s in range(W):
        pool = torch.randn(cap, 2, hkv, 16, 128, generator=g, device=dev).to(torch.bfloat16)
        insts.append(DcpInstance(ctx, W, s, hq, hkv, cap, kv_pool=pool, n_max=64, m_max=64))
    for s in range(W):
        for t in range(W):
            insts[s].set_peer_local(t, insts[t])
        insts[s].commit()
    active = list(range(len(lens)))
    # one decode step with the new token written by K8 before attention
    pl.append_many(active)
    pl.build_routing()
    for s in range(W):
        v = pl.instance_view(s)
        mids = device_to_numpy(v.m_ids, v.m_rows, np.int64)
        if len(mids):
            kv = torch.randn(len(mids), 2, hkv, 128, generator=g, device=dev).to(torch.bfloat16)
            pl.kv_append(s, kv, [x.kv_pool for x in insts])
    q = {i: torch.randn(hq, 128, generator=g, device=dev).to(torch.bfloat16) for i in active}
    out, views = run_local_step(pl, insts, q)
    port = oracle_lib.port()
    partial = {}
    for s in range(W):
        v = views[s]
        n = v.n_rows
        cu = device_to_numpy(v.cu_pages, n + 1, np.int32)
        nid = device_to_numpy(v.n_ids, n, np.int64)
        b = workload.PagedBatch(device_to_numpy(v.shard_len, n, np.int64), cu,
                                device_to_numpy(v.block_table, int(cu[-1]), np.int32), cap, hq, hkv)
        fill = device_to_numpy(v.page_fill, int(cu[-1]), np.uint8)
        o, l = oracle_lib.paged_decode_f64(b, _bits(torch.stack([q[int(r)] for r in nid])),
                                           _bits(insts[s].kv_pool), fill)
        for j, r in enumerate(nid):
            partial[(int(r), s)] = (o[j], l[j])
    for r in active:
        p = pl.placement(r)
        tot = sum(int(device_to_numpy(views[s].shard_len, views[s].n_rows, np.int64)[
            list(device_to_numpy(views[s].n_ids, views[s].n_rows, np.int64)).index(r)]) for s in p["kv"])
        assert tot == lens[r] + 1                      # the appended token is attended
        for h in range(hq):
            ro, rl = _oracle_merge(port, [partial[(r, s)][0][h] for s in p["kv"]],
                                   [partial[(r, s)][1][h] for s in p["kv"]], 128)
            o = out[r][0][h].astype(np.float64)
            assert np.linalg.norm(o - ro) / np.linalg.norm(ro) <= 2e-2
            assert abs(float(out[r][1][h]) - rl) <= 1e-5 * max(1.0, abs(rl))
