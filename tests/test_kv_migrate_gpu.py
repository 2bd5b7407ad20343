"""Prefill -> decode KV migration (MIGRATE / TRANSFER).

After the planner admits requests (GlobalPageTable::allocate, page_table.cpp:9-49),
dcp_kv_migrate copies each request's contiguous prefill K / V into the frames of
its page table, on every instance of its KV binding.  Checked two ways:

* bytes: every logical page of the compiled reference's own page table (the CSV of
  dcpsim_ref::GlobalPageTable::dump_csv for the same script) holds exactly the
  request's tokens of that page, kv_binding member by member; frames the table
  does not list stay untouched;
* end to end: a routed DCP step (K2 -> K1 -> K3) over the migrated pools equals the
  reference's sharded_attention_merge (attn_merge.cpp:64-77) over the contiguous
  prefill KV with bounds = the placement's splits — bf16 at rel-L2 <= 2e-2, fp32 at
  SPEC.md:380's 1e-5.
"""
import numpy as np
import pytest
import torch

from tests import oracle_lib
from paper_2605_21100_b200._capi import device_to_numpy

pytestmark = pytest.mark.gpu
I64MAX = 2**63 - 1
BUCKET = [[40, 1], [2000, 2], [I64MAX, 4]]
LENS = [5000, 37, 1500, 700, 12000, 1, 16, 17, 33, 4096]


def _setup(dtype, cap=400, W=4, hkv=8):
    from paper_2605_21100_b200.attention import DcpContext
    from paper_2605_21100_b200.planner import DevicePlanner
    ctx = DcpContext(0)
    dev = torch.device("cuda:0")
    pl = DevicePlanner(ctx, 1, W, 16, cap, "dcp", BUCKET, max_requests=64)
    ids = list(range(len(LENS)))
    pl.enqueue_many(ids, LENS)
    assert pl.step()["committed"] == ids
    g = torch.Generator(device=dev).manual_seed(11)
    src_k = [torch.randn(L, hkv, 128, generator=g, device=dev).to(dtype) for L in LENS]
    src_v = [torch.randn(L, hkv, 128, generator=g, device=dev).to(dtype) for L in LENS]
    pools = [torch.zeros(cap, 2, hkv, 16, 128, dtype=dtype, device=dev) for _ in range(W)]
    pl.migrate_kv(ids, src_k, src_v, pools)
    torch.cuda.synchronize()
    return ctx, pl, ids, src_k, src_v, pools


def _reference_table(W, cap):
    ref = oracle_lib.World(oracle_lib.reference(), "dcpref_", 1, W, 16, cap, "dcp", BUCKET)
    for i, L in enumerate(LENS):
        ref.enqueue(i, L)
    ref.step()
    return ref


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_migrate_matches_reference_page_table(dtype):
    W, cap = 4, 400
    ctx, pl, ids, src_k, src_v, pools = _setup(dtype, cap, W)
    ref = _reference_table(W, cap)
    assert pl.page_table_csv() == ref.page_table_csv()
    rows = [list(map(int, l.split(","))) for l in ref.page_table_csv().strip().split("\n")[1:]]
    host = [p.cpu() for p in pools]
    touched = [set() for _ in range(W)]
    tok = {}
    for rid, page, inst, frame in rows:
        p = ref.placement(rid)
        # tokens of logical page `page`: members in kv_binding order, ceil(split/16) pages each
        t0, left = None, page
        acc = 0
        for sp in p["split"]:
            np_ = -(-sp // 16)
            if left < np_:
                t0 = acc + 16 * left
                fill = min(16, sp - 16 * left)
                break
            left -= np_
            acc += sp
        assert t0 is not None
        tok[rid] = tok.get(rid, 0) + fill
        k = src_k[rid][t0:t0 + fill].cpu().transpose(0, 1)   # [hkv, fill, d]
        v = src_v[rid][t0:t0 + fill].cpu().transpose(0, 1)
        assert torch.equal(host[inst][frame, 0, :, :fill], k), (rid, page)
        assert torch.equal(host[inst][frame, 1, :, :fill], v), (rid, page)
        touched[inst].add(frame)
    assert tok == {i: L for i, L in enumerate(LENS)}
    for s in range(W):
        rest = [f for f in range(cap) if f not in touched[s]]
        assert not host[s][rest].any(), s


@pytest.mark.parametrize("dtype,tol", [(torch.bfloat16, 2e-2), (torch.float32, 1e-5)])
def test_migrated_step_equals_sharded_attention_merge(dtype, tol):
    from paper_2605_21100_b200.dcp_step import DcpInstance, run_local_step
    W, cap, hq, hkv = 4, 400, 32, 8
    ctx, pl, ids, src_k, src_v, pools = _setup(dtype, cap, W, hkv)
    dname = "bf16" if dtype == torch.bfloat16 else "f32"
    insts = [DcpInstance(ctx, W, s, hq, hkv, cap, kv_pool=pools[s], n_max=64, m_max=64, dtype=dname)
             for s in range(W)]
    for s in range(W):
        for t in range(W):
            insts[s].set_peer_local(t, insts[t])
        insts[s].commit()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(12)
    q = {i: torch.randn(hq, 128, generator=g, device=dev).to(dtype) for i in ids}
    out, _ = run_local_step(pl, insts, q)
    R = oracle_lib.reference()
    P = oracle_lib.P
    G = hq // hkv
    worst = 0.0
    for rid in ids:
        split = pl.placement(rid)["split"]
        bounds = np.cumsum(np.array(split, np.int64))
        assert bounds[-1] == LENS[rid]
        K = src_k[rid].float().cpu().double().numpy()
        V = src_v[rid].float().cpu().double().numpy()
        Q = q[rid].float().cpu().double().numpy()
        for h in range(hq):
            kh = np.ascontiguousarray(K[:, h // G])
            vh = np.ascontiguousarray(V[:, h // G])
            o = np.zeros(128)
            rc = R.dcpref_sharded_attention_merge_f64(P(np.ascontiguousarray(Q[h])), P(kh), P(vh), LENS[rid], 128,
                                                      1.0 / np.sqrt(128.0), P(bounds), len(bounds), 0, P(o))
            assert rc == 0
            got = out[rid][0][h].astype(np.float64)
            rel = np.linalg.norm(got - o) / np.linalg.norm(o)
            worst = max(worst, rel)
    print(f"migrated DCP step vs sharded_attention_merge ({dname}): worst rel-L2 {worst:.2e}")
    assert worst <= tol, worst
