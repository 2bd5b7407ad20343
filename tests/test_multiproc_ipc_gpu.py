"""Two processes, one instance each, exchanging through CUDA-IPC-mapped peer pools.

The first execution of the multi-process path (dcp_xchg_open_peer_ipc / dcp_moe_open_peer_ipc,
system-scope flags between processes): two ranks on cuda:0 (gpurun provides one GPU; CUDA IPC
between processes on the same device is the same mechanism as across NVLink), gloo for the
handle all-gather and the planner-replica digest, nothing else on the host between the ranks.
Each rank runs three consecutive decode steps of
    K2 -> K1 (+ Res-route) -> K3          (DCP attention, one CP-2 request across both ranks)
    K4 -> K5a (region) -> experts -> K5b -> K5c   (MoE over K7's device M count)
with no phase ordering: every cross-rank wait is a device flag (the driver time-slices the two
contexts).  Each rank checks its own M rows against the fp64 oracles.
"""
import os
import queue
import socket
import time
import traceback

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

I64MAX = 2**63 - 1
W, HQ, HKV, CAP = 2, 32, 8, 700
LENS = [5000, 300, 2048, 17, 1, 4096, 900]
BUCKET = [[1000, 1], [I64MAX, 2]]
MOE = dict(hidden=1024, experts=8, topk=2, m_max=16)
FFN = 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pool(rank, cap, hkv):
    import torch
    g = torch.Generator().manual_seed(100 + rank)
    return torch.randn(cap, 2, hkv, 16, 128, generator=g).to(torch.bfloat16)


def _q(rid, step):
    import torch
    g = torch.Generator().manual_seed(1000 * step + rid)
    return torch.randn(HQ, 128, generator=g).to(torch.bfloat16)


def _tok(rid, step, H, E, k):
    import torch
    g = torch.Generator().manual_seed(7000 + 1000 * step + rid)
    x = torch.randn(H, generator=g).to(torch.bfloat16)
    top = torch.topk(torch.randn(E, generator=g), k)
    return x, top.indices.to(torch.int32), torch.softmax(top.values, -1).float()


def _weights():
    import torch
    g = torch.Generator().manual_seed(55)
    H, E = MOE["hidden"], MOE["experts"]
    wg = (torch.randn(E, FFN, H, generator=g) / H ** 0.5).to(torch.bfloat16)
    wu = (torch.randn(E, FFN, H, generator=g) / H ** 0.5).to(torch.bfloat16)
    wd = (torch.randn(E, H, FFN, generator=g) / FFN ** 0.5).to(torch.bfloat16)
    return wg, wu, wd


def _worker(rank, port, q, log_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import faulthandler
    import sys
    if log_dir:  # per-rank log with a stack dump if the rank is still running after 240 s
        f = open(os.path.join(log_dir, f"ipc_rank{rank}.log"), "w", buffering=1)
        sys.stdout = sys.stderr = f
        faulthandler.enable(f)
        faulthandler.dump_traceback_later(240, exit=False, file=f)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=W)
    try:
        from paper_2605_21100_b200 import workload
        from paper_2605_21100_b200._capi import device_to_numpy
        from paper_2605_21100_b200.attention import DcpContext
        from paper_2605_21100_b200.multi import RankStep
        from tests import oracle_lib
        from tests.test_dcp_step_gpu import _bits, _oracle_merge
        from tests.test_exchange_protocol_gpu import _expert_rows
        dev = torch.device("cuda:0")
        ctx = DcpContext(0)
        rs = RankStep(ctx, W, rank, LENS, HQ, HKV, CAP, lambda r, c, h: _pool(r, c, h).to(dev), bucket=BUCKET,
                      moe=MOE, timeout_ms=60000, n_max=64, m_max=32)
        pl = rs.planner
        assert any(len(pl.placement(r)["kv"]) == 2 for r in rs.ids)
        H, E, k = MOE["hidden"], MOE["experts"], MOE["topk"]
        wg, wu, wd = _weights()
        per = E // W
        wgd, wud, wdd = (w[rank * per:(rank + 1) * per].to(dev) for w in (wg, wu, wd))

        def experts(xr, mr, counts, y):
            for src in range(W):
                n = int(counts[src])
                if n:
                    y[src, :n] = _expert_rows(xr[src, :n], mr[src, :n], rank * per, wgd, wud, wdd)

        port_lib = oracle_lib.port()
        P = oracle_lib.P
        # oracle partials need every instance's pool and page lists: rebuild both (deterministic)
        views = [pl.instance_view(s) for s in range(W)]
        pools = [_pool(s, CAP, HKV) for s in range(W)]
        worst_o = worst_l = worst_moe = 0.0
        for step in range(3):
            qrows = torch.stack([_q(r, step) for r in rs.m_ids]).to(dev) if rs.m_ids else None
            rs.attention(qrows)
            toks = [_tok(r, step, H, E, k) for r in rs.m_ids]
            x = torch.stack([t[0] for t in toks]).to(dev)
            idx = torch.stack([t[1] for t in toks]).contiguous().to(dev)
            wts = torch.stack([t[2] for t in toks]).contiguous().to(dev)
            rs.moe_layer(x, idx, wts, expert_fn=experts)
            torch.cuda.synchronize()
            rs.status()
            o, l = rs.results()
            partial = {}
            for s in range(W):
                v = views[s]
                n = v.n_rows
                cu = device_to_numpy(v.cu_pages, n + 1, np.int32)
                nid = device_to_numpy(v.n_ids, n, np.int64)
                b = workload.PagedBatch(device_to_numpy(v.shard_len, n, np.int64), cu,
                                        device_to_numpy(v.block_table, int(cu[-1]), np.int32), CAP, HQ, HKV)
                fill = device_to_numpy(v.page_fill, int(cu[-1]), np.uint8)
                qs = torch.stack([_q(int(r), step) for r in nid])
                po, plse = oracle_lib.paged_decode_f64(b, _bits(qs), _bits(pools[s]), fill)
                for j, r in enumerate(nid):
                    partial[(int(r), s)] = (po[j], plse[j])
            for j, r in enumerate(rs.m_ids):
                kv = pl.placement(r)["kv"]
                for h in range(HQ):
                    ro, rl = _oracle_merge(port_lib, [partial[(r, s)][0][h] for s in kv],
                                           [partial[(r, s)][1][h] for s in kv], 128)
                    worst_o = max(worst_o, np.linalg.norm(o[j][h] - ro) / np.linalg.norm(ro))
                    worst_l = max(worst_l, abs(float(l[j][h]) - rl) / max(1.0, abs(rl)))
            M = len(rs.m_ids)
            ref = np.zeros((M, H))
            assert port_lib.dcpora_moe_layer_f64(M, H, FFN, E, k, P(_bits(x.cpu())), P(idx.cpu().numpy()),
                                                 P(wts.cpu().numpy()), P(_bits(wg)), P(_bits(wu)), P(_bits(wd)),
                                                 P(ref), 8) == 0
            got = rs.moe.out[:M].cpu().double().numpy()
            worst_moe = max(worst_moe, (np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)).max())
        assert worst_o <= 2e-2 and worst_l <= 1e-5 and worst_moe <= 2e-2, (worst_o, worst_l, worst_moe)
        q.put((rank, "ok", len(rs.m_ids), worst_o, worst_l, worst_moe))
        import datetime
        dist.monitored_barrier(timeout=datetime.timedelta(seconds=300))  # the peer still maps our pools
        rs.close()
    except Exception:
        q.put((rank, traceback.format_exc(), 0, 0, 0, 0))
    finally:
        dist.destroy_process_group()


def _graph_worker(rank, port, q, log_dir):
    """Whole-layer graph replay across processes: step 0 eager, steps 1-3 replayed from each
    rank's dcp_layer_graph (K7 of its planner replica inside), bit-identical to step 0."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    if log_dir:
        f = open(os.path.join(log_dir, f"ipc_graph_rank{rank}.log"), "w", buffering=1)
        sys.stdout = sys.stderr = f
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=W)
    try:
        from paper_2605_21100_b200.attention import DcpContext
        from paper_2605_21100_b200.dcp_step import LayerGraph
        from paper_2605_21100_b200.multi import RankStep
        dev = torch.device("cuda:0")
        ctx = DcpContext(0)
        rs = RankStep(ctx, W, rank, LENS, HQ, HKV, CAP, lambda r, c, h: _pool(r, c, h).to(dev), bucket=BUCKET,
                      moe=MOE, timeout_ms=60000, n_max=64, m_max=32)
        H, E, k = MOE["hidden"], MOE["experts"], MOE["topk"]
        M = len(rs.m_ids)
        mm = MOE["m_max"]
        xb = torch.zeros(mm, H, dtype=torch.bfloat16, device=dev)
        ib = torch.zeros(mm, k, dtype=torch.int32, device=dev)
        wb = torch.zeros(mm, k, dtype=torch.float32, device=dev)
        if M:
            toks = [_tok(r, 0, H, E, k) for r in rs.m_ids]
            xb[:M] = torch.stack([t[0] for t in toks]).to(dev)
            ib[:M] = torch.stack([t[1] for t in toks]).to(dev)
            wb[:M] = torch.stack([t[2] for t in toks]).to(dev)
            rs.inst.write_queries(torch.stack([_q(r, 0) for r in rs.m_ids]).to(dev))
        rs.inst.run(rs.view)
        rs.moe_layer(xb[:M], ib[:M], wb[:M])
        torch.cuda.synchronize()
        rs.status()
        o0, l0 = (a.copy() for a in rs.results())
        m0 = rs.moe.out[:M].cpu().numpy().copy()
        g = LayerGraph(rs.inst, rs.view, rs.moe, xb, ib, wb, planner=rs.planner)
        for step in range(3):
            g.launch(M)
            torch.cuda.synchronize()
            rs.status()
            o, l = rs.results()
            assert np.array_equal(o, o0) and np.array_equal(l, l0), f"attention differs at replay {step}"
            assert np.array_equal(rs.moe.out[:M].cpu().numpy(), m0), f"MoE differs at replay {step}"
        # the one-launch step (dcp_decode_step_fused): eager, then inside a fused layer graph
        for step in range(2):
            rs.inst.run(rs.view, None, "fused")
            torch.cuda.synchronize()
            rs.status()
            o, l = rs.results()
            assert np.array_equal(o, o0) and np.array_equal(l, l0), f"fused step {step} differs"
        # K5b + K5c in one launch (dcp_moe_combine_fused), eager: bit-identical to the two launches;
        # and K4 + K5a in one launch (dcp_moe_step_dispatch_recv): the whole MoE layer in 2 launches
        for step in range(3):
            rs.moe_layer(xb[:M], ib[:M], wb[:M], fused_combine=True, fused_receive=step > 0)
            torch.cuda.synchronize()
            rs.status()
            assert np.array_equal(rs.moe.out[:M].cpu().numpy(), m0), f"fused MoE layer {step} differs"
        gf = LayerGraph(rs.inst, rs.view, rs.moe, xb, ib, wb, planner=rs.planner, fused=True)
        for step in range(3):
            gf.launch(M)
            torch.cuda.synchronize()
            rs.status()
            o, l = rs.results()
            assert np.array_equal(o, o0) and np.array_equal(l, l0), f"fused graph replay {step} differs"
            assert np.array_equal(rs.moe.out[:M].cpu().numpy(), m0), f"MoE differs at fused replay {step}"
        q.put((rank, "ok", M, g.info()["graphs"], 0, 0))
        import datetime
        dist.monitored_barrier(timeout=datetime.timedelta(seconds=300))
        g.close()
        gf.close()
        rs.close()
    except Exception:
        q.put((rank, traceback.format_exc(), 0, 0, 0, 0))
    finally:
        dist.destroy_process_group()


def _spawn(target):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    log_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(log_dir, exist_ok=True)
    procs = [ctx.Process(target=target, args=(r, port, q, log_dir)) for r in range(W)]
    for p in procs:
        p.start()
    res = []
    deadline = time.time() + 600
    while len(res) < W and time.time() < deadline:
        try:
            res.append(q.get(timeout=5))
        except queue.Empty:
            dead = [(i, p.exitcode) for i, p in enumerate(procs) if p.exitcode not in (None, 0)]
            assert not dead, f"rank(s) died without a result: {dead} (see gpurun_out/ipc_rank*.log)"
    for p in procs:
        p.join(timeout=120)
        if p.exitcode is None:
            p.kill()
    assert len(res) == W, f"only {len(res)} of {W} ranks reported: {res} (see gpurun_out/ipc_rank*.log)"
    res.sort()
    for rank, msg, *_ in res:
        assert msg == "ok", f"rank {rank}:\n{msg}"
    for p in procs:
        assert p.exitcode == 0
    return res


def test_two_processes_ipc_dcp_and_moe():
    res = _spawn(_worker)
    for rank, msg, m, wo, wl, wm in res:
        print(f"rank {rank}: {m} M rows, 3 steps: O rel-L2 {wo:.2e}, LSE {wl:.2e}, MoE {wm:.2e}")
    assert sum(r[2] for r in res) == len(LENS)


def test_two_processes_layer_graph_replay():
    res = _spawn(_graph_worker)
    for rank, msg, m, n_graphs, *_ in res:
        print(f"rank {rank}: {m} M rows, {n_graphs} layer graphs, 3 replays bit-identical to the eager step")
    assert sum(r[2] for r in res) == len(LENS)
