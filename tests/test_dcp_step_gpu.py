"""A full routed DCP decode step (K6 -> K7 -> K2 -> K1+Res-route -> K3) on W
instances hosted on one GPU, checked against the oracle.

Oracle per request r: for every s in P_r (kv_binding order) the reference
shard_attention<double> (attn_merge.hpp:53-82) over r's tokens on s, then
lse_merge (attn_merge.hpp:86-100) over the non-empty shards — i.e. the
reference's sharded_attention_merge semantics (attn_merge.cpp:35-46) with the
per-instance token sets the device page table produced.
"""
import numpy as np
import pytest
import torch

from tests import oracle_lib
from paper_2605_21100_b200 import workload
from paper_2605_21100_b200._capi import device_to_numpy

pytestmark = pytest.mark.gpu
I64MAX = 2**63 - 1


def _bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def _oracle_merge(port, outs, lses, d):
    live = [i for i in range(len(lses)) if np.isfinite(lses[i])]
    o = np.zeros(d)
    P = oracle_lib.P
    oo = np.ascontiguousarray(np.stack([outs[i] for i in live]))
    ll = np.ascontiguousarray(np.array([lses[i] for i in live], np.float64))
    assert port.dcpora_lse_merge_f64(len(live), P(oo), P(ll), d, P(o)) == 0
    m = ll.max()
    return o, m + np.log(np.exp(ll - m).sum())


@pytest.mark.parametrize("hq,hkv,W,policy", [(32, 8, 4, "dcp"), (32, 4, 2, "dcp"), (32, 8, 4, "uniform")])
def test_routed_step_matches_oracle(hq, hkv, W, policy):
    from paper_2605_21100_b200.attention import DcpContext
    from paper_2605_21100_b200.dcp_step import DcpInstance, run_local_step
    from paper_2605_21100_b200.planner import DevicePlanner
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    cap = 1200
    bucket = [[1500, 1], [6000, 2], [I64MAX, 4]]
    pl = DevicePlanner(ctx, 1, W, 16, cap, policy, bucket, uniform_degree=2, hol_strict=False,
                       max_requests=256)
    rng = np.random.default_rng(5 + W)
    ids = list(range(30))
    lens = [int(x) for x in rng.integers(1, 3000 * W, size=30)]
    pl.enqueue_many(ids, lens)
    pl.step()
    active = [i for i in ids if pl.placement(i) is not None]
    for rid in rng.choice(active, 40).tolist():      # decode growth -> partial pages
        pl.append_token(rid)
    pl.step()                                         # rebalance moves m_r
    active = [i for i in ids if pl.placement(i) is not None]
    assert len(active) >= 5
    g = torch.Generator(device=dev).manual_seed(7)
    insts = []
    for s in range(W):
        pool = torch.randn(cap, 2, hkv, 16, 128, generator=g, device=dev).to(torch.bfloat16)
        insts.append(DcpInstance(ctx, W, s, hq, hkv, cap, kv_pool=pool, n_max=256, m_max=256))
    for s in range(W):
        for t in range(W):
            insts[s].set_peer_local(t, insts[t])
        insts[s].commit()
    q = {i: torch.randn(hq, 128, generator=g, device=dev).to(torch.bfloat16) for i in active}
    res, views = run_local_step(pl, insts, q)
    assert sorted(res) == sorted(active)

    # oracle: per-instance shard partials from the device page table's block tables
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
        b = workload.PagedBatch(sl, cu, bt, cap, hq, hkv)
        qs = torch.stack([q[int(r)] for r in nid]) if n else torch.zeros(0, hq, 128, dtype=torch.bfloat16)
        o, l = oracle_lib.paged_decode_f64(b, _bits(qs), _bits(insts[s].kv_pool), fill)
        for j, r in enumerate(nid):
            partial[(int(r), s)] = (o[j], l[j])
    worst_o, worst_l = 0.0, 0.0
    for r in active:
        p = pl.placement(r)
        for h in range(hq):
            outs = [partial[(r, s)][0][h] for s in p["kv"]]
            lses = [partial[(r, s)][1][h] for s in p["kv"]]
            ro, rl = _oracle_merge(port, outs, lses, 128)
            o, l = res[r][0][h].astype(np.float64), float(res[r][1][h])
            worst_o = max(worst_o, np.linalg.norm(o - ro) / np.linalg.norm(ro))
            worst_l = max(worst_l, abs(l - rl) / max(1.0, abs(rl)))
    assert worst_o <= 2e-2, worst_o
    assert worst_l <= 1e-5, worst_l
    # at least one request really was split across instances (CP > 1)
    assert any(len(pl.placement(r)["kv"]) > 1 for r in active)
