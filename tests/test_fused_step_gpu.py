"""One launch per routed step (dcp_decode_step_fused; VERDICT r1 "routed small-step floor").

The fused launch folds begin_step (fence + epoch), K2's Q-route puts (prologue) and K3's LSE
merges (epilogue) into K1.  It must equal the four phased calls bit for bit, keep the epoch
protocol intact when fused and phased steps alternate (both parities), and work inside the
whole-layer graph.  W = 1 here (every producer is co-resident); the multi-process case is in
tests/test_multiproc_ipc_gpu.py.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _one(lens, cap=6000):
    from paper_2605_21100_b200.attention import DcpContext
    from paper_2605_21100_b200.dcp_step import DcpInstance
    from paper_2605_21100_b200.planner import DevicePlanner
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    pl = DevicePlanner(ctx, 1, 1, 16, cap, "dcp", None, max_requests=512, reserve_pages=8)
    pl.enqueue_many(list(range(len(lens))), lens)
    assert len(pl.step()["committed"]) == len(lens)
    pl.build_routing()
    g = torch.Generator(device=dev).manual_seed(21)
    pool = torch.randn(cap, 2, 8, 16, 128, generator=g, device=dev).to(torch.bfloat16)
    inst = DcpInstance(ctx, 1, 0, 32, 8, cap, kv_pool=pool, n_max=512, m_max=256)
    inst.set_peer_local(0, inst)
    inst.commit()
    v = pl.instance_view(0)
    inst.write_queries(torch.randn(v.m_rows, 32, 128, generator=g, device=dev).to(torch.bfloat16))
    return ctx, pl, inst, v


def _res(inst, v):
    torch.cuda.synchronize()
    inst.status()
    o, l = inst.results(v.m_rows)
    return o.copy(), l.copy()


@pytest.mark.parametrize("lens", [[1000] * 16, [100] * 4, [1, 17, 4096, 300, 2500, 16, 33, 70000],
                                  list(range(1, 200, 7))])
def test_fused_equals_phased_across_parities(lens):
    ctx, pl, inst, v = _one(lens)
    inst.run(v, None, "all")
    ref = _res(inst, v)
    for phase in ("fused", "fused", "all", "fused", "all", "all", "fused"):
        inst.run(v, None, phase)
        o, l = _res(inst, v)
        assert np.array_equal(o, ref[0]) and np.array_equal(l, ref[1]), phase


def test_fused_layer_graph_equals_eager():
    from paper_2605_21100_b200.dcp_step import LayerGraph
    from paper_2605_21100_b200.moe import MoeInstance
    ctx, pl, inst, v = _one([300, 17, 4000, 1, 2500, 900, 64, 1000])
    dev = torch.device("cuda:0")
    moe = MoeInstance(ctx, 1, 0, 512, 2, 8, 256)
    moe.set_peer_local(0, moe)
    moe.commit()
    g = torch.Generator(device=dev).manual_seed(4)
    x = torch.randn(256, 512, generator=g, device=dev).to(torch.bfloat16)
    top = torch.topk(torch.randn(256, 8, generator=g, device=dev), 2, dim=-1)
    idx, w = top.indices.to(torch.int32).contiguous(), torch.softmax(top.values, -1).float().contiguous()
    inst.run(v, None, "all")
    y = torch.zeros(1, 256, 512, dtype=torch.bfloat16, device=dev)
    M = v.m_rows
    moe.dispatch(x[:M], idx[:M], w[:M], m_count_ptr=v.m_count_all)
    moe.receive_regions()
    moe.expert_identity(y)
    moe.combine_put_regions(y)
    moe.combine_reduce()
    ref = _res(inst, v)
    mref = moe.out[:M].cpu().numpy().copy()
    lg = LayerGraph(inst, v, moe, x, idx, w, planner=pl, fused=True)
    for _ in range(3):
        lg.launch(M)
        o, l = _res(inst, v)
        moe.status()
        assert np.array_equal(o, ref[0]) and np.array_equal(l, ref[1])
        assert np.array_equal(moe.out[:M].cpu().numpy(), mref)
    lg.close()
