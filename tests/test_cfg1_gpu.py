"""BASELINE.json configs[0] (cfg1) end to end on the device path.

One node of 2 instances, make_cluster capacity 1,024 pages of 16 tokens; 8 requests with
lengths uniform_int(mt19937_64(1), 128, 4096); BucketFn {1024 -> 1, INT64_MAX -> 2}, so the
longer requests take CP 2 (the cfg1 variant SURVEY §8(d) asks for); MHA 8 q = 8 kv heads,
d = 128; MoE with 4 experts top-2, hidden 1,024, expert FFN 256.  cfg1 is fp32 (the
reference's production precision, attn_merge.cpp:64-77), and so is the device path here:
fp32 KV / Q through K1-f32 and the fp32 exchange (q_elem_bytes 4).

Checked, each against the oracle:
- K6 / K7: the page-table and routing CSVs equal the oracle port's, byte for byte;
- K2 + K1-f32 + K3: every request's merged O / LSE vs shard_attention<double> + lse_merge over
  the device page table's per-instance tokens, at SPEC.md:380's fp32 bar (rel-L2 <= 1e-5,
  LSE <= 1e-5 * max(1, |lse|));
- K4 / K5: each instance's 8-token decode batch through dispatch -> experts -> combine vs
  dcpora_moe_layer_f64 (rel-L2 <= 2e-2 per token).
"""
import numpy as np
import pytest
import torch

from tests import oracle_lib
from tests.oracle_lib import World
from tests.test_dcp_step_gpu import _bits, _oracle_merge
from paper_2605_21100_b200 import workload
from paper_2605_21100_b200._capi import device_to_numpy

pytestmark = pytest.mark.gpu
I64MAX = 2**63 - 1
W, HQ, HKV, D, PAGE, CAP = 2, 8, 8, 128, 16, 1024
BUCKET = [[1024, 1], [I64MAX, 2]]


def test_cfg1_planner_attention_moe():
    from paper_2605_21100_b200.attention import DcpContext
    from paper_2605_21100_b200.dcp_step import DcpInstance, run_local_step
    from paper_2605_21100_b200.moe import MoeInstance
    from paper_2605_21100_b200.planner import DevicePlanner
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    lens = workload.lengths(1, 8, 128, 4096)
    ids = list(range(8))

    # ---- planner (K6) and routing (K7) vs the oracle port
    pl = DevicePlanner(ctx, 1, W, PAGE, CAP, "dcp", BUCKET, max_requests=64)
    ow = World(oracle_lib.port(), "dcpora_", 1, W, PAGE, CAP, "dcp", BUCKET)
    pl.enqueue_many(ids, lens)
    for i, L in zip(ids, lens):
        ow.enqueue(i, L)
    assert pl.step() == ow.step()
    assert pl.page_table_csv() == ow.page_table_csv()
    assert pl.routing_csv() == ow.routing_csv()
    active = [i for i in ids if pl.placement(i) is not None]
    assert len(active) == 8
    assert any(len(pl.placement(r)["kv"]) == 2 for r in active)  # CP 2 under the cfg1 bucket

    # ---- routed fp32 attention step (K2 -> K1-f32 + Res-route -> K3) vs the fp64 oracle
    g = torch.Generator(device=dev).manual_seed(2)
    insts = []
    for s in range(W):
        pool = torch.randn(CAP, 2, HKV, PAGE, D, generator=g, device=dev)
        insts.append(DcpInstance(ctx, W, s, HQ, HKV, CAP, kv_pool=pool, n_max=64, m_max=64, dtype="f32"))
    for s in range(W):
        for t in range(W):
            insts[s].set_peer_local(t, insts[t])
        insts[s].commit()
    q = {i: torch.randn(HQ, D, generator=g, device=dev) for i in active}
    res, views = run_local_step(pl, insts, q)
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
        b = workload.PagedBatch(sl, cu, bt, CAP, HQ, HKV)
        qs = torch.stack([q[int(r)] for r in nid]).cpu().numpy() if n else np.zeros((0, HQ, D), np.float32)
        o, l = oracle_lib.paged_decode_f32in_f64(b, qs, insts[s].kv_pool.cpu().numpy(), fill)
        for j, r in enumerate(nid):
            partial[(int(r), s)] = (o[j], l[j])
    worst_o = worst_l = 0.0
    for r in active:
        p = pl.placement(r)
        for h in range(HQ):
            ro, rl = _oracle_merge(port, [partial[(r, s)][0][h] for s in p["kv"]],
                                   [partial[(r, s)][1][h] for s in p["kv"]], D)
            o, l = res[r][0][h].astype(np.float64), float(res[r][1][h])
            worst_o = max(worst_o, np.linalg.norm(o - ro) / np.linalg.norm(ro))
            worst_l = max(worst_l, abs(l - rl) / max(1.0, abs(rl)))
    print(f"cfg1 fp32 routed step: worst O rel-L2 {worst_o:.3e}, LSE {worst_l:.3e}")
    assert worst_o <= 1e-5, worst_o
    assert worst_l <= 1e-5, worst_l

    # ---- MoE layer on each instance's MoE-bound decode tokens (K4 -> experts -> K5)
    E, k, H, I = 4, 2, 1024, 256
    homes = [[r for r in active if pl.placement(r)["moe"] == s] for s in range(W)]
    moe = [MoeInstance(ctx, W, s, H, k, E, 16) for s in range(W)]
    for s in range(W):
        for t in range(W):
            moe[s].set_peer_local(t, moe[t])
        moe[s].commit()
    w_gate = (torch.randn(E, I, H, generator=g, device=dev) / H ** 0.5).to(torch.bfloat16)
    w_up = (torch.randn(E, I, H, generator=g, device=dev) / H ** 0.5).to(torch.bfloat16)
    w_down = (torch.randn(E, H, I, generator=g, device=dev) / I ** 0.5).to(torch.bfloat16)
    toks = []
    for s in range(W):
        M = len(homes[s])
        x = torch.randn(M, H, generator=g, device=dev).to(torch.bfloat16)
        top = torch.topk(torch.randn(M, E, generator=g, device=dev), k, dim=-1)
        toks.append((x, top.indices.to(torch.int32).contiguous(),
                     torch.softmax(top.values, dim=-1).float().contiguous()))
    for s in range(W):
        moe[s].dispatch(*toks[s])
    rows = [moe[s].receive() for s in range(W)]
    per = E // W
    for s in range(W):
        moe[s].expert_stage(rows[s][0], w_gate[s * per:(s + 1) * per], w_up[s * per:(s + 1) * per],
                            w_down[s * per:(s + 1) * per])
    for s in range(W):
        moe[s].combine_put()
    for s in range(W):
        moe[s].combine_reduce()
    torch.cuda.synchronize()
    P = oracle_lib.P
    worst = 0.0
    for s in range(W):
        x, idx, wts = toks[s]
        M = x.shape[0]
        if M == 0:
            continue
        ref = np.zeros((M, H))
        assert port.dcpora_moe_layer_f64(M, H, I, E, k, P(_bits(x)), P(idx.cpu().numpy()), P(wts.cpu().numpy()),
                                         P(_bits(w_gate)), P(_bits(w_up)), P(_bits(w_down)), P(ref), 8) == 0
        got = moe[s].out[:M].cpu().double().numpy()
        worst = max(worst, (np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)).max())
    assert worst <= 2e-2, worst
    for x in insts + moe:
        x.close()
    pl.close()
