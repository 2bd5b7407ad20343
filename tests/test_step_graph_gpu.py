"""AOT step graphs (dcp_step_graph_*): the captured routed step replays with
per-step metadata from the device planner and matches the eager path bit for
bit across decode steps (growth, re-planning) and bucket changes.  One
instance (all routes local): a single GPU cannot host several instances'
whole-step graphs on one stream, since each instance's K1 waits on the other
instances' Q-route puts."""
import numpy as np
import pytest
import torch

from paper_2605_21100_b200._capi import device_to_numpy

pytestmark = pytest.mark.gpu


def test_graph_replay_matches_eager():
    from paper_2605_21100_b200.attention import DcpContext
    from paper_2605_21100_b200.dcp_step import DcpInstance, StepGraph
    from paper_2605_21100_b200.planner import DevicePlanner
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    cap = 3000
    pl = DevicePlanner(ctx, 1, 1, 16, cap, "dcp", None, max_requests=512, reserve_pages=32)
    g = torch.Generator(device=dev).manual_seed(4)
    pool = torch.randn(cap, 2, 8, 16, 128, generator=g, device=dev).to(torch.bfloat16)
    eager = DcpInstance(ctx, 1, 0, 32, 8, cap, kv_pool=pool, n_max=512, m_max=256)
    graphd = DcpInstance(ctx, 1, 0, 32, 8, cap, kv_pool=pool, n_max=512, m_max=256)
    for x in (eager, graphd):
        x.set_peer_local(0, x)
        x.commit()
    rng = np.random.default_rng(0)
    ids = list(range(40))
    lens = rng.integers(1, 1500, size=40).tolist()
    pl.enqueue_many(ids[:10], lens[:10])
    pl.step()
    pl.build_routing()
    view = pl.instance_view(0)
    sg = StepGraph(graphd, view)
    assert sg.graphs == 6 and sg.buckets == 48
    q = {i: torch.randn(32, 128, generator=g, device=dev).to(torch.bfloat16) for i in ids}
    nxt = 10
    for step in range(12):
        if step in (3, 7):                      # new arrivals change M (bucket switch)
            pl.enqueue_many(ids[nxt:nxt + 15], lens[nxt:nxt + 15])
            nxt += 15
            pl.step()
        active = [i for i in ids[:nxt] if pl.placement(i) is not None]
        pl.append_many(active)
        pl.build_routing()
        v = pl.instance_view(0)
        m_ids = device_to_numpy(v.m_ids, v.m_rows, np.int64)
        qs = torch.stack([q[int(i)] for i in m_ids])
        eager.write_queries(qs)
        graphd.write_queries(qs)
        eager.run(v)
        sg.launch(v.m_rows, v.n_rows)
        torch.cuda.synchronize()
        o1, l1 = eager.results(v.m_rows)
        o2, l2 = graphd.results(v.m_rows)
        assert np.array_equal(o1, o2) and np.array_equal(l1, l2), step
        assert np.all(np.isfinite(o1))
