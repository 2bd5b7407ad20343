"""K10 MLA split-KV paged decode attention (tcgen05 CTA pairs) vs the CPU oracle.

Oracle: dcpora_mla_paged_decode_f64 = shard_attention<double> (attn_merge.hpp:53-82)
per (shard, head) with keys = the 576-wide cache rows and values = their first
512 columns, over exactly-widened bf16 inputs.  The reference does not model MLA
(SPEC.md:381), so this restatement is the checker.
Tolerances (north_star bf16 bar): O rel-L2 <= 2e-2 per (shard, head) vector;
LSE |d| <= 2e-4 * max(1, |lse|).
"""
import numpy as np
import pytest
import torch

from tests import oracle_lib
from paper_2605_21100_b200 import workload

pytestmark = pytest.mark.gpu

O_TOL = 2e-2
LSE_TOL = 2e-4
DK = 576


@pytest.fixture(scope="module")
def ctx():
    from paper_2605_21100_b200.attention import DcpContext
    assert torch.cuda.is_available(), "GPU test selected but no CUDA device"
    return DcpContext(0)


def _bits(t):
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def _case(lens, page=16, seed=0, frame_order="shuffled", spare=7):
    b = workload.paged_batch(lens, 128, 1, DK, page, frame_order=frame_order, seed=seed, spare_frames=spare)
    g = torch.Generator().manual_seed(seed + 1)
    q = torch.randn(len(lens), 128, DK, generator=g).to(torch.bfloat16)
    pool = torch.randn(b.num_frames, page, DK, generator=g).to(torch.bfloat16)
    return b, q, pool


def _run(ctx, b, q, pool, page_fill=None, att=None, reps=1):
    from paper_2605_21100_b200.attention import MlaDecodeAttention
    dev = torch.device("cuda:0")
    att = att or MlaDecodeAttention(ctx, b.page_size, max_shards=max(len(b.shard_len), 1))
    pf = torch.from_numpy(page_fill).to(dev) if page_fill is not None else None
    args = (q.to(dev), pool.to(dev), torch.from_numpy(b.block_table).to(dev),
            torch.from_numpy(b.cu_pages).to(dev), torch.from_numpy(b.shard_len).to(dev))
    for _ in range(reps):
        out, lse = att(*args, page_fill=pf)
    torch.cuda.synchronize()
    return out.cpu().double().numpy(), lse.cpu().double().numpy()


def _check(b, q, pool, out, lse, page_fill=None):
    ro, rl = oracle_lib.mla_decode_f64(b, _bits(q), _bits(pool), page_fill)
    ne = b.shard_len > 0
    assert np.all(np.isneginf(lse[~ne])) and np.all(out[~ne] == 0.0)
    rel = np.linalg.norm(out[ne] - ro[ne], axis=-1) / np.linalg.norm(ro[ne], axis=-1)
    dl = np.abs(lse[ne] - rl[ne]) / np.maximum(1.0, np.abs(rl[ne]))
    assert np.isfinite(out[ne]).all() and np.isfinite(lse[ne]).all()
    assert rel.max() <= O_TOL, f"O rel-L2 {rel.max():.3e} at {np.unravel_index(rel.argmax(), rel.shape)}"
    assert dl.max() <= LSE_TOL, f"LSE |d| {dl.max():.3e} at {np.unravel_index(dl.argmax(), dl.shape)}"
    return rel.max(), dl.max()


def test_mla_edges(ctx):
    """Tails, an empty shard, single tokens, more pairs than tiles (T < pairs)."""
    b, q, pool = _case([1, 17, 128, 129, 300, 0, 1000, 4096])
    out, lse = _run(ctx, b, q, pool)
    _check(b, q, pool, out, lse)


def test_mla_stream_k(ctx):
    """Many tiles per pair; shards cut across pairs and merged by the last finisher."""
    lens = workload.lengths(5, 12, 1024, 24576)
    b, q, pool = _case(lens, seed=5)
    out, lse = _run(ctx, b, q, pool, reps=2)  # second launch checks the re-armed counters
    _check(b, q, pool, out, lse)


def test_mla_skewed(ctx):
    """One long shard among short ones: stream-K splits the long one over most pairs."""
    b, q, pool = _case([65536 + 37, 200, 3000, 1], seed=9)
    out, lse = _run(ctx, b, q, pool)
    _check(b, q, pool, out, lse)


def test_mla_page_fill(ctx):
    """Partially filled non-final pages (append_token fallback, page_table.cpp:104-113)."""
    rng = np.random.default_rng(3)
    lens = [700, 33, 2048]
    pages = [(n + 15) // 16 for n in lens]
    fill = []
    for n, pg in zip(lens, pages):
        f = np.full(pg, 16, np.uint8)
        f[-1] = n - 16 * (pg - 1)
        holes = rng.choice(pg, size=max(1, pg // 5), replace=False)
        f[holes] = rng.integers(1, 16, size=len(holes))
        fill.append(f)
    fill = np.concatenate(fill)
    b, q, pool = _case(lens, seed=11)
    cu = b.cu_pages
    b.shard_len[:] = [int(fill[cu[i]:cu[i + 1]].sum()) for i in range(len(lens))]
    out, lse = _run(ctx, b, q, pool, page_fill=fill)
    _check(b, q, pool, out, lse, page_fill=fill)


@pytest.mark.parametrize("page", [32, 64])
def test_mla_page_sizes(ctx, page):
    b, q, pool = _case([1, 100, 2000, 5000], page=page, seed=page)
    out, lse = _run(ctx, b, q, pool)
    _check(b, q, pool, out, lse)


def test_mla_many_shards(ctx):
    """1,100 shards (the tile scan's carry across 1,024-shard chunks), mostly 1-3 tiles each,
    zero-token shards interleaved, several segments per pair."""
    rng = np.random.default_rng(21)
    lens = rng.integers(1, 400, size=1100)
    lens[::97] = 0
    b, q, pool = _case(lens.tolist(), seed=21, spare=3)
    out, lse = _run(ctx, b, q, pool)
    _check(b, q, pool, out, lse)


@pytest.mark.parametrize("W", [4, 8])
def test_mla_routed_dcp_step(ctx, W):
    """cfg5-shaped DCP attention split across W instances (one GPU, same code path as across
    GPUs): K6 -> K7 -> K2 (576-wide Q rows) -> K10 routed (Q-route flag waits, O / LSE into
    m_r's 512-wide result slots) -> K3, two consecutive steps; every request and head against
    shard_attention<double> on each instance's tokens + lse_merge (bf16 bar)."""
    from paper_2605_21100_b200._capi import device_to_numpy
    from paper_2605_21100_b200.dcp_step import MlaDcpInstance, run_local_step
    from paper_2605_21100_b200.planner import DevicePlanner
    from tests.test_dcp_step_gpu import _oracle_merge
    I64MAX = 2**63 - 1
    dev = torch.device("cuda:0")
    cap = 3000
    pl = DevicePlanner(ctx, 1, W, 16, cap, "dcp", [[3000, 1], [20000, 2], [I64MAX, W]], max_requests=64)
    rng = np.random.default_rng(W)
    lens = [90000, 25000, 17, 1, 4000] + rng.integers(1, 6000, size=10).tolist()
    pl.enqueue_many(list(range(len(lens))), lens)
    assert len(pl.step()["committed"]) == len(lens)
    assert len(pl.placement(0)["kv"]) == W
    g = torch.Generator(device=dev).manual_seed(9)
    insts = []
    for s in range(W):
        pool = torch.randn(cap, 16, DK, generator=g, device=dev).to(torch.bfloat16)
        insts.append(MlaDcpInstance(ctx, W, s, cap, kv_pool=pool, n_max=64, m_max=32))
    for s in range(W):
        for t in range(W):
            insts[s].set_peer_local(t, insts[t])
        insts[s].commit()
    port = oracle_lib.port()
    active = list(range(len(lens)))
    for step in range(2):
        q = {i: torch.randn(128, DK, generator=g, device=dev).to(torch.bfloat16) for i in active}
        res, views = run_local_step(pl, insts, q)
        partial = {}
        for s in range(W):
            v = views[s]
            n = v.n_rows
            cu = device_to_numpy(v.cu_pages, n + 1, np.int32)
            nid = device_to_numpy(v.n_ids, n, np.int64)
            b = workload.PagedBatch(device_to_numpy(v.shard_len, n, np.int64), cu,
                                    device_to_numpy(v.block_table, int(cu[-1]), np.int32), cap, 128, 1, DK, 16)
            fill = device_to_numpy(v.page_fill, int(cu[-1]), np.uint8)
            qs = torch.stack([q[int(r)] for r in nid]).cpu()
            o, l = oracle_lib.mla_decode_f64(b, _bits(qs), _bits(insts[s].kv_pool.cpu()), fill)
            for j, r in enumerate(nid):
                partial[(int(r), s)] = (o[j], l[j])
        worst_o = worst_l = 0.0
        for r in active:
            kv = pl.placement(r)["kv"]
            for h in range(128):
                ro, rl = _oracle_merge(port, [partial[(r, s)][0][h] for s in kv],
                                       [partial[(r, s)][1][h] for s in kv], 512)
                o = res[r][0][h].astype(np.float64)
                worst_o = max(worst_o, np.linalg.norm(o - ro) / np.linalg.norm(ro))
                worst_l = max(worst_l, abs(float(res[r][1][h]) - rl) / max(1.0, abs(rl)))
        print(f"MLA routed W={W} step {step}: worst O rel-L2 {worst_o:.3e}, LSE {worst_l:.3e}")
        assert worst_o <= O_TOL, worst_o
        assert worst_l <= LSE_TOL, worst_l
        pl.append_many(active)
    for x in insts:
        x.close()
    pl.close()


@pytest.mark.parametrize("name", ["cfg2-shaped (64 req, KV 1K-32K)", "long-mix (1 x 512K + 63 x 1K-8K)"])
def test_mla_bench_inputs_all_shards(ctx, name):
    """bench_mla.py's own workloads at full size (the K10 numbers in bench.py's line): every
    shard and head of the bench's seeded pool and queries against the fp64 oracle."""
    import bench_mla
    from paper_2605_21100_b200.attention import MlaDecodeAttention
    dev = torch.device("cuda:0")
    lens = bench_mla.workloads()[name]
    b, pool, q = bench_mla.inputs(dev, lens)
    att = MlaDecodeAttention(ctx, b.page_size, max_shards=len(lens))
    out, lse = att(q, pool, torch.from_numpy(b.block_table).to(dev), torch.from_numpy(b.cu_pages).to(dev),
                   torch.from_numpy(b.shard_len).to(dev))
    torch.cuda.synchronize()
    rel, dl = _check(b, q.cpu(), pool.cpu(), out.cpu().double().numpy(), lse.cpu().double().numpy())
    print(f"{name}: {len(lens)} shards x 128 heads, worst O rel-L2 {rel:.3e}, LSE |d| {dl:.3e}")


def test_mla_graph_replay(ctx):
    """K10's three launches (tile scan -> decode -> merge, PDL-chained) captured in a CUDA graph
    and replayed: bit-identical to the eager call."""
    from paper_2605_21100_b200.attention import MlaDecodeAttention
    dev = torch.device("cuda:0")
    b, q, pool = _case(workload.lengths(3, 24, 200, 9000), seed=31)
    att = MlaDecodeAttention(ctx, b.page_size, max_shards=len(b.shard_len))
    out, lse = att.prepare(q.to(dev), pool.to(dev), torch.from_numpy(b.block_table).to(dev),
                           torch.from_numpy(b.cu_pages).to(dev), torch.from_numpy(b.shard_len).to(dev))
    att.launch()
    torch.cuda.synchronize()
    o0, l0 = out.clone(), lse.clone()
    out.zero_()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            att.launch(st)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, o0) and torch.equal(lse, l0)
    _check(b, q, pool, out.cpu().double().numpy(), lse.cpu().double().numpy())
