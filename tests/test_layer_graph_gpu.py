"""Whole-layer AOT decode graphs (Alg. 2, 805-840).

dcp_layer_graph captures one instance's decode layer — [K7] -> K2 -> K1 -> K3 -> K4 -> expert
-> K5 — per (M-bucket, MoE parity).  Replays must equal the eager calls bit for bit:

* W = 1 with K7 inside the graph, over several replays (both parities), plus a replay after
  the planner state changed (append_token): the in-graph K7 sees the new lengths;
* several instances each replaying their own graph: tests/test_multiproc_ipc_gpu.py (one
  process per instance — instances sharing one GPU inside one process cannot run whole-layer
  graphs concurrently: a K1 spinning on a peer's Q-route occupies every SM the peer needs);
* an expert-stage callback (captured cudaMemcpyAsync of the parity's receive region) gets
  the right region pointer on both parities;
* the MoE output against the numpy definition of the gate-weighted identity expert.
"""
import ctypes
import glob
import os

import numpy as np
import pytest
import torch

from paper_2605_21100_b200._capi import device_to_numpy

pytestmark = pytest.mark.gpu
I64MAX = 2**63 - 1
H, E, K = 512, 16, 4


def _cudart():
    import torch as _t
    p = glob.glob(os.path.join(os.path.dirname(_t.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
    L = ctypes.CDLL(p[0] if p else "libcudart.so")
    L.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    L.cudaMemcpyAsync.restype = ctypes.c_int
    return L


def _world(W, lens, bucket=None, cap=2000):
    from paper_2605_21100_b200.attention import DcpContext
    from paper_2605_21100_b200.dcp_step import DcpInstance
    from paper_2605_21100_b200.moe import MoeInstance
    from paper_2605_21100_b200.planner import DevicePlanner
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    pl = DevicePlanner(ctx, 1, W, 16, cap, "dcp", bucket, max_requests=256, reserve_pages=16)
    pl.enqueue_many(list(range(len(lens))), lens)
    assert len(pl.step()["committed"]) == len(lens)
    pl.build_routing()
    g = torch.Generator(device=dev).manual_seed(3)
    insts, moes = [], []
    for s in range(W):
        pool = torch.randn(cap, 2, 8, 16, 128, generator=g, device=dev).to(torch.bfloat16)
        insts.append(DcpInstance(ctx, W, s, 32, 8, cap, kv_pool=pool, n_max=128, m_max=64))
        moes.append(MoeInstance(ctx, W, s, H, K, E, 64))
    for s in range(W):
        for t in range(W):
            insts[s].set_peer_local(t, insts[t])
            moes[s].set_peer_local(t, moes[t])
        insts[s].commit()
        moes[s].commit()
    views = [pl.instance_view(s) for s in range(W)]
    bufs = []
    for s in range(W):
        M = views[s].m_rows
        q = torch.randn(max(M, 1), 32, 128, generator=g, device=dev).to(torch.bfloat16)[:M]
        if M:
            insts[s].write_queries(q)
        x = torch.randn(64, H, generator=g, device=dev).to(torch.bfloat16)
        top = torch.topk(torch.randn(64, E, generator=g, device=dev), K, dim=-1)
        idx = top.indices.to(torch.int32).contiguous()
        w = torch.softmax(top.values, -1).float().contiguous()
        bufs.append((x, idx, w))
    return ctx, pl, insts, moes, views, bufs


def _eager(insts, moes, views, bufs):
    W = len(insts)
    for s in range(W):
        insts[s].run(views[s], None, "q")
    for s in range(W):
        insts[s].run(views[s], None, "attn")
    for s in range(W):
        insts[s].run(views[s], None, "merge")
    ys = []
    for s in range(W):
        x, idx, w = bufs[s]
        moes[s].dispatch(x, idx, w, m_count_ptr=views[s].m_count_all + 4 * s)
    for s in range(W):
        moes[s].receive_regions()
    for s in range(W):
        y = torch.zeros(W, 64, H, dtype=torch.bfloat16, device=x.device)
        moes[s].expert_identity(y)
        ys.append(y)
    for s in range(W):
        moes[s].combine_put_regions(ys[s])
    for s in range(W):
        moes[s].combine_reduce()
    torch.cuda.synchronize()
    return _snap(insts, moes, views)


def _snap(insts, moes, views):
    for i in insts:
        i.status()
    for m in moes:
        m.status()
    out = []
    for s, inst in enumerate(insts):
        o, l = inst.results(views[s].m_rows)
        out.append((o.copy(), l.copy(), moes[s].out[:views[s].m_rows].cpu().numpy().copy()))
    return out


def _same(a, b):
    for (o1, l1, m1), (o2, l2, m2) in zip(a, b):
        assert np.array_equal(o1, o2) and np.array_equal(l1, l2) and np.array_equal(m1, m2)


def _moe_reference(bufs, views):
    """out_t = sum over t's distinct expert ranks of bf16((sum of that rank's gate weights) * x_t)."""
    W = len(bufs)
    for s in range(W):
        x, idx, w = (t.cpu() for t in bufs[s])
        M = views[s].m_rows
        ref = np.zeros((M, H), np.float32)
        for t in range(M):
            for d in range(W):
                sel = (idx[t] // (E // W)) == d
                if sel.any():
                    ws = float(w[t][sel].sum())
                    ref[t] += (x[t].float() * ws).to(torch.bfloat16).float().numpy()
        yield s, ref


def test_layer_graph_w1_k7_inside_matches_eager():
    from paper_2605_21100_b200.dcp_step import LayerGraph
    lens = [300, 17, 4000, 1, 2500, 900, 64, 1000]
    ctx, pl, insts, moes, views, bufs = _world(1, lens)
    ref = _eager(insts, moes, views, bufs)
    x, idx, w = bufs[0]
    g = LayerGraph(insts[0], views[0], moes[0], x, idx, w, planner=pl)
    info = g.info()
    assert info["graphs"] == 2 * info["buckets"] and info["buckets"] == 4  # M-hat 8, 16, 32, 64
    for _ in range(3):  # both parities
        g.launch(views[0].m_rows)
        torch.cuda.synchronize()
        _same(ref, _snap(insts, moes, views))
    # the planner state moves on: every request grows by one token; the in-graph K7 re-derives
    # the block tables and shard lengths, so the replay equals eager routing + step
    pl.append_many(list(range(len(lens))))
    g.launch(views[0].m_rows)
    torch.cuda.synchronize()
    got = _snap(insts, moes, views)
    pl.build_routing()
    ref2 = _eager(insts, moes, views, bufs)
    _same(ref2, got)
    assert not np.array_equal(ref[0][0], got[0][0])  # the appended tokens changed the attention
    for s, r in _moe_reference(bufs, views):
        np.testing.assert_allclose(got[s][2], r, rtol=1e-2, atol=1e-2)
    g.close()


def test_layer_graph_expert_callback_gets_parity_regions():
    from paper_2605_21100_b200 import _capi
    from paper_2605_21100_b200.dcp_step import LayerGraph
    rt = _cudart()
    lens = [700, 33, 1200, 5]
    Wn = 1
    ctx, pl, insts, moes, views, bufs = _world(Wn, lens)
    calls = []

    def copy_expert(user, stream, parity, x_region, meta, counts, y_region):
        calls.append(parity)
        rc = rt.cudaMemcpyAsync(y_region, x_region, Wn * 64 * H * 2, 3, stream)  # D2D
        assert rc == 0

    cb = _capi.EXPERT_FN(copy_expert)
    graphs = [LayerGraph(insts[s], views[s], moes[s], *bufs[s], expert=cb) for s in range(Wn)]
    nb = graphs[0].info()["buckets"]
    assert sorted(calls) == [0] * (Wn * nb) + [1] * (Wn * nb)
    streams = [torch.cuda.Stream() for _ in range(Wn)]
    for step in range(3):
        for s in range(Wn):  # a fresh token batch every step: a stale parity would return old rows
            x, idx, w = bufs[s]
            x.copy_(torch.randn_like(x, dtype=torch.float32).to(torch.bfloat16))
        torch.cuda.synchronize()
        for s in range(Wn):
            graphs[s].launch(views[s].m_rows, streams[s])
        torch.cuda.synchronize()
        for s in range(Wn):
            moes[s].status()
            x, idx, _ = (t.cpu() for t in bufs[s])
            M = views[s].m_rows
            nranks = np.array([len(set((idx[t] // (E // Wn)).tolist())) for t in range(M)], np.float32)
            want = x[:M].float().numpy() * nranks[:, None]
            np.testing.assert_allclose(moes[s].out[:M].cpu().numpy(), want, rtol=1e-2, atol=1e-2)
    for g in graphs:
        g.close()
