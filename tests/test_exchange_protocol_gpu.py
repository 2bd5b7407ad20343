"""The exchange step protocol (exchange.cuh): epoch-parity double buffers, the begin_step
fence, bounded flag waits with an error word, for the DCP exchange (K2/K1/K3) and the MoE
exchange (K4/K5).  W instances on one GPU through the same code path as across GPUs.

* consecutive routed steps with fresh queries alternate the parity buffers and each step
  matches the oracle;
* a peer that never begins a step makes the fence time out: DCP_E_TIMEOUT, not a hang;
* a partial that never arrives makes K3 time out the same way;
* the MoE region path (rows read in place from the pool) over consecutive steps matches the
  expert oracle, and K4's count records agree with the gating.
"""
import time

import numpy as np
import pytest
import torch

from tests import oracle_lib
from tests.test_dcp_step_gpu import _bits, _oracle_merge
from paper_2605_21100_b200 import workload
from paper_2605_21100_b200._capi import ExchangeTimeout, device_to_numpy

pytestmark = pytest.mark.gpu
I64MAX = 2**63 - 1


def _ctx():
    from paper_2605_21100_b200.attention import DcpContext
    return DcpContext(0)


def _instances(ctx, W, hq, hkv, cap, g, timeout_ms=0, dtype="bf16"):
    from paper_2605_21100_b200.dcp_step import DcpInstance
    dev = torch.device("cuda:0")
    insts = []
    for s in range(W):
        pool = torch.randn(cap, 2, hkv, 16, 128, generator=g, device=dev)
        if dtype == "bf16":
            pool = pool.to(torch.bfloat16)
        insts.append(DcpInstance(ctx, W, s, hq, hkv, cap, kv_pool=pool, n_max=128, m_max=128,
                                 timeout_ms=timeout_ms, dtype=dtype))
    for s in range(W):
        for t in range(W):
            insts[s].set_peer_local(t, insts[t])
        insts[s].commit()
    return insts


def _oracle_step(pl, insts, views, q, active, hq, cap):
    port = oracle_lib.port()
    partial = {}
    for s, inst in enumerate(insts):
        v = views[s]
        n = v.n_rows
        cu = device_to_numpy(v.cu_pages, n + 1, np.int32)
        nid = device_to_numpy(v.n_ids, n, np.int64)
        b = workload.PagedBatch(device_to_numpy(v.shard_len, n, np.int64), cu,
                                device_to_numpy(v.block_table, int(cu[-1]), np.int32), cap, hq, inst.hkv)
        fill = device_to_numpy(v.page_fill, int(cu[-1]), np.uint8)
        qs = torch.stack([q[int(r)] for r in nid]) if n else torch.zeros(0, hq, 128, dtype=torch.bfloat16)
        o, l = oracle_lib.paged_decode_f64(b, _bits(qs), _bits(inst.kv_pool), fill)
        for j, r in enumerate(nid):
            partial[(int(r), s)] = (o[j], l[j])
    out = {}
    for r in active:
        p = pl.placement(r)
        out[r] = [_oracle_merge(port, [partial[(r, s)][0][h] for s in p["kv"]],
                                [partial[(r, s)][1][h] for s in p["kv"]], 128) for h in range(hq)]
    return out


def test_consecutive_steps_alternate_parity():
    """Five routed steps with fresh queries (parities 1, 0, 1, 0, 1) and decode growth between
    them; every step's merged outputs match the oracle, so no step read another's slots."""
    from paper_2605_21100_b200.dcp_step import run_local_step
    from paper_2605_21100_b200.planner import DevicePlanner
    ctx = _ctx()
    dev = torch.device("cuda:0")
    W, hq, hkv, cap = 4, 32, 8, 800
    pl = DevicePlanner(ctx, 1, W, 16, cap, "dcp", [[1000, 1], [4000, 2], [I64MAX, 4]], max_requests=64,
                       reserve_pages=8)
    rng = np.random.default_rng(1)
    ids = list(range(20))
    pl.enqueue_many(ids, [int(x) for x in rng.integers(1, 9000, size=20)])
    pl.step()
    active = [i for i in ids if pl.placement(i) is not None]
    g = torch.Generator(device=dev).manual_seed(4)
    insts = _instances(ctx, W, hq, hkv, cap, g)
    for step in range(5):
        q = {i: torch.randn(hq, 128, generator=g, device=dev).to(torch.bfloat16) for i in active}
        res, views = run_local_step(pl, insts, q)
        ref = _oracle_step(pl, insts, views, q, active, hq, cap)
        for r in active:
            for h in range(hq):
                ro, rl = ref[r][h]
                o = res[r][0][h].astype(np.float64)
                assert np.linalg.norm(o - ro) / np.linalg.norm(ro) <= 2e-2, (step, r, h)
                assert abs(float(res[r][1][h]) - rl) <= 1e-5 * max(1.0, abs(rl)), (step, r, h)
        pl.append_many(active)           # the next step sees one more token per request
    for x in insts:
        x.close()
    pl.close()


def test_fence_times_out_when_a_peer_never_steps():
    """Instance 0 begins three steps while instance 1 begins none: the third begin_step needs
    instance 1 to have begun step 2 and times out -> DCP_E_TIMEOUT with the fence site."""
    from paper_2605_21100_b200 import _capi
    import ctypes
    ctx = _ctx()
    g = torch.Generator(device="cuda:0").manual_seed(0)
    insts = _instances(ctx, 2, 8, 8, 8, g, timeout_ms=200)
    L = _capi.lib()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    t0 = time.time()
    for _ in range(3):
        _capi.check(L.dcp_xchg_begin_step(insts[0].x, s))
    info = (ctypes.c_uint32 * 4)()
    rc = L.dcp_xchg_status(insts[0].x, info)
    assert rc == -11, rc
    assert info[1] >> 24 == 1 and (info[1] >> 16) & 0xff == 1   # SITE_FENCE, peer 1
    assert info[2] == 1                                          # wanted done >= 1
    assert time.time() - t0 < 20
    insts[0].status()                      # the error word was cleared
    assert torch.ones(4, device="cuda:0").sum().item() == 4      # the GPU is alive


def test_merge_times_out_when_a_partial_never_arrives():
    """A CP-2 request whose second shard's instance never runs its attention: K3 at the MoE
    binding waits for that partial, times out, and the step reports ExchangeTimeout."""
    from paper_2605_21100_b200.planner import DevicePlanner
    ctx = _ctx()
    dev = torch.device("cuda:0")
    W, hq, hkv, cap = 2, 8, 8, 64
    pl = DevicePlanner(ctx, 1, W, 16, cap, "dcp", [[100, 1], [I64MAX, 2]], max_requests=8)
    pl.enqueue_many([0], [500])
    pl.step()
    assert len(pl.placement(0)["kv"]) == 2
    pl.build_routing()
    g = torch.Generator(device=dev).manual_seed(1)
    insts = _instances(ctx, W, hq, hkv, cap, g, timeout_ms=200)
    views = [pl.instance_view(s) for s in range(W)]
    m = pl.placement(0)["moe"]
    insts[m].write_queries(torch.randn(1, hq, 128, generator=g, device=dev).to(torch.bfloat16))
    for s in range(W):
        insts[s].run(views[s], phase="q")
    insts[m].run(views[m], phase="attn")       # the other instance never runs its shard
    insts[m].run(views[m], phase="merge")
    with pytest.raises(ExchangeTimeout):
        insts[m].status()
    for x in insts:
        x.close()
    pl.close()


def _expert_rows(x, meta, e0, w_gate, w_up, w_down):
    """Library-GEMM expert FFN of received rows (x bf16 [R, H], meta int32 [R, meta])."""
    R, H = x.shape
    y = torch.zeros(R, H, dtype=torch.float32, device=x.device)
    m = meta.cpu().numpy()
    per = {}
    for r in range(R):
        for j in range(int(m[r, 1])):
            per.setdefault(int(m[r, 2 + 2 * j]), []).append((r, float(np.int32(m[r, 3 + 2 * j]).view(np.float32))))
    for e in sorted(per):
        rows = torch.tensor([r for r, _ in per[e]], device=x.device)
        wts = torch.tensor([w for _, w in per[e]], device=x.device, dtype=torch.float32)
        xe = x[rows]
        a = (torch.nn.functional.silu((xe @ w_gate[e - e0].T).float()) * (xe @ w_up[e - e0].T).float())
        y.index_add_(0, rows, (a.to(torch.bfloat16) @ w_down[e - e0].T).float() * wts[:, None])
    return y.to(torch.bfloat16)


@pytest.mark.parametrize("W,E,k,H,I,M", [(4, 16, 4, 1024, 64, 48), (8, 64, 8, 2048, 32, 128)])
def test_moe_region_path_consecutive_steps(W, E, k, H, I, M):
    """K4 -> K5a (region mode) -> experts reading the pool in place -> K5b (region) -> K5c,
    three steps in a row with fresh tokens and M from a device counter."""
    from paper_2605_21100_b200.moe import MoeInstance
    ctx = _ctx()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(E + W)
    inst = [MoeInstance(ctx, W, s, H, k, E, M) for s in range(W)]
    for s in range(W):
        for t in range(W):
            inst[s].set_peer_local(t, inst[t])
        inst[s].commit()
    w_gate = (torch.randn(E, I, H, generator=g, device=dev) / H ** 0.5).to(torch.bfloat16)
    w_up = (torch.randn(E, I, H, generator=g, device=dev) / H ** 0.5).to(torch.bfloat16)
    w_down = (torch.randn(E, H, I, generator=g, device=dev) / I ** 0.5).to(torch.bfloat16)
    per = E // W
    port = oracle_lib.port()
    P = oracle_lib.P
    y_region = [torch.zeros(W, M, H, dtype=torch.bfloat16, device=dev) for _ in range(W)]
    for step in range(3):
        toks = []
        for s in range(W):
            Ms = M - 7 * s if step != 1 or s != 2 else 0
            x = torch.randn(Ms, H, generator=g, device=dev).to(torch.bfloat16)
            top = torch.topk(torch.randn(Ms, E, generator=g, device=dev), k, dim=-1)
            toks.append((x, top.indices.to(torch.int32).contiguous(), torch.softmax(top.values, -1).float().contiguous()))
        mcnt = [torch.tensor([t[0].shape[0]], dtype=torch.int32, device=dev) for t in toks]
        for s in range(W):
            inst[s].dispatch(*toks[s], m_count_ptr=mcnt[s].data_ptr())
        for s in range(W):
            inst[s].receive_regions()
        for s in range(W):
            xr, mr = inst[s].regions()
            cnt = inst[s].recv_counts()
            expect = [int(((toks[src][1] // per) == s).any(dim=1).sum().item()) for src in range(W)]
            assert cnt.tolist() == expect, (step, s)
            for src in range(W):
                n = int(cnt[src])
                if n:
                    y_region[s][src, :n] = _expert_rows(xr[src, :n], mr[src, :n], s * per, w_gate[s * per:(s + 1) * per],
                                                        w_up[s * per:(s + 1) * per], w_down[s * per:(s + 1) * per])
        for s in range(W):
            inst[s].combine_put_regions(y_region[s])
        for s in range(W):
            inst[s].combine_reduce()
        torch.cuda.synchronize()
        for s in range(W):
            inst[s].status()
        worst = 0.0
        for s in range(W):
            x, idx, wts = toks[s]
            Ms = x.shape[0]
            if Ms == 0:
                continue
            ref = np.zeros((Ms, H))
            assert port.dcpora_moe_layer_f64(Ms, H, I, E, k, P(_bits(x)), P(idx.cpu().numpy()), P(wts.cpu().numpy()),
                                             P(_bits(w_gate)), P(_bits(w_up)), P(_bits(w_down)), P(ref), 8) == 0
            got = inst[s].out[:Ms].cpu().double().numpy()
            worst = max(worst, (np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)).max())
        assert worst <= 2e-2, (step, worst)
    for i in inst:
        i.close()
