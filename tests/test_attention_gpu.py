"""K1+K9 split-KV paged decode attention vs the CPU oracle (GPU parity tests).

Oracle: dcpora_paged_decode_attn_f64 = shard_attention<double>
(attn_merge.hpp:53-82) per (shard, q-head) over exactly-widened bf16 inputs.
Tolerances (north_star / SURVEY §7.2a): bf16 path O rel-L2 <= 2e-2 per
(shard, head) vector; LSE |d| <= 1e-5 * max(1, |lse|).
"""
import math

import numpy as np
import pytest
import torch

from tests import oracle_lib
from paper_2605_21100_b200 import workload

pytestmark = pytest.mark.gpu

O_TOL = 2e-2
LSE_TOL = 1e-5


@pytest.fixture(scope="module")
def ctx():
    from paper_2605_21100_b200.attention import DcpContext
    assert torch.cuda.is_available(), "GPU test selected but no CUDA device"
    return DcpContext(0)


def _make(batch, seed, fill_variant=None):
    g = torch.Generator().manual_seed(seed)
    R, hq, hkv, d, page = (len(batch.shard_len), batch.num_q_heads, batch.num_kv_heads,
                           batch.head_dim, batch.page_size)
    q = torch.randn(R, hq, d, generator=g).to(torch.bfloat16)
    pool = torch.randn(batch.num_frames, 2, hkv, page, d, generator=g).to(torch.bfloat16)
    return q, pool


def _run(ctx, batch, q, pool, page_fill=None, scale=None):
    from paper_2605_21100_b200.attention import DecodeAttention
    dev = torch.device("cuda:0")
    att = DecodeAttention(ctx, batch.num_q_heads, batch.num_kv_heads, batch.head_dim,
                          batch.page_size, max_shards=max(len(batch.shard_len), 1))
    pf = torch.from_numpy(page_fill).to(dev) if page_fill is not None else None
    out, lse = att(q.to(dev), pool.to(dev), torch.from_numpy(batch.block_table).to(dev),
                   torch.from_numpy(batch.cu_pages).to(dev), torch.from_numpy(batch.shard_len).to(dev),
                   page_fill=pf, scale=scale)
    torch.cuda.synchronize()
    return out.cpu().double().numpy(), lse.cpu().double().numpy(), att


def _bits(t):
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def _check(batch, q, pool, out, lse, page_fill=None, scale=None):
    ref_o, ref_l = oracle_lib.paged_decode_f64(batch, _bits(q), _bits(pool), page_fill, scale)
    nonempty = batch.shard_len > 0
    # zero-token shards: O = 0, LSE = -inf
    assert np.all(np.isneginf(lse[~nonempty])), "empty shard LSE must be -inf"
    assert np.all(out[~nonempty] == 0)
    o, r = out[nonempty], ref_o[nonempty]
    rel = np.linalg.norm(o - r, axis=-1) / np.maximum(np.linalg.norm(r, axis=-1), 1e-30)
    assert rel.max() <= O_TOL, f"O rel-L2 {rel.max():.3e}"
    dl = np.abs(lse[nonempty] - ref_l[nonempty])
    bound = LSE_TOL * np.maximum(1.0, np.abs(ref_l[nonempty]))
    assert np.all(dl <= bound), f"LSE max |d| {dl.max():.3e}"
    return rel.max(), dl.max()


@pytest.mark.parametrize("hq,hkv", [(32, 8), (32, 4), (8, 8), (32, 2), (16, 1)])
def test_small_shapes(ctx, hq, hkv):
    lens = [1, 15, 16, 17, 33, 200, 0, 1000, 4097]
    b = workload.paged_batch(lens, hq, hkv, frame_order="shuffled", seed=1, spare_frames=37)
    q, pool = _make(b, 1)
    out, lse, _ = _run(ctx, b, q, pool)
    _check(b, q, pool, out, lse)


@pytest.mark.parametrize("page", [32, 64])
@pytest.mark.parametrize("hq,hkv", [(32, 8), (32, 4)])
def test_page_sizes(ctx, hq, hkv, page):
    # ClusterTopology::page_size (types.hpp:92) other than 16: split ring, 16-token chunks
    rng = np.random.default_rng(page + hkv)
    lens = [1, 15, 16, 17, page - 1, page, page + 1, 0] + rng.integers(1, 5000, size=12).tolist()
    b = workload.paged_batch(lens, hq, hkv, page_size=page, frame_order="shuffled", seed=5, spare_frames=9)
    q, pool = _make(b, 12)
    out, lse, _ = _run(ctx, b, q, pool)
    _check(b, q, pool, out, lse)
    # per-page fills, incl. a non-final partial page and a page holding < 16 tokens
    fill = np.full(int(b.cu_pages[-1]), page, np.uint8)
    for r, L in enumerate(lens):
        if b.cu_pages[r + 1] > b.cu_pages[r]:
            fill[b.cu_pages[r + 1] - 1] = L - page * (b.cu_pages[r + 1] - b.cu_pages[r] - 1)
    big = int(np.argmax(lens))
    fill[b.cu_pages[big]] = 3
    fill[b.cu_pages[big] + 1] = page - 7
    out, lse, _ = _run(ctx, b, q, pool, page_fill=fill)
    _check(b, q, pool, out, lse, page_fill=fill)


def test_cross_cta_splits(ctx):
    # enough pages that most shards are cut by several of the 148 page ranges
    rng = np.random.default_rng(7)
    lens = rng.integers(1, 6000, size=24).tolist() + [0, 0, 3]
    b = workload.paged_batch(lens, 32, 8, frame_order="shuffled", seed=2, spare_frames=100)
    q, pool = _make(b, 2)
    out, lse, _ = _run(ctx, b, q, pool)
    _check(b, q, pool, out, lse)


def test_tiny_grid_underfilled(ctx):
    # fewer pages than CTAs: most CTAs own an empty range
    b = workload.paged_batch([5, 40, 0, 16], 32, 8)
    q, pool = _make(b, 3)
    out, lse, _ = _run(ctx, b, q, pool)
    _check(b, q, pool, out, lse)


def test_page_fill_non_final_partial(ctx):
    # append_token's fallback can leave a non-final partial page
    # (page_table.cpp:101-113): per-page fill counts.
    lens = [46, 300, 77]
    b = workload.paged_batch(lens, 32, 8, frame_order="shuffled", seed=4, spare_frames=5)
    fill = np.full(int(b.cu_pages[-1]), 16, np.uint8)
    for r, L in enumerate(lens):
        fill[b.cu_pages[r + 1] - 1] = L - 16 * (b.cu_pages[r + 1] - b.cu_pages[r] - 1)
    fill[1] = 14                     # request 0: 16, 14, 14 — a non-final partial page
    fill[b.cu_pages[1] + 3] = 9      # request 1: partial page in the middle
    fill[b.cu_pages[2]] = 1          # request 2: single-token first page
    q, pool = _make(b, 4)
    out, lse, _ = _run(ctx, b, q, pool, page_fill=fill)
    _check(b, q, pool, out, lse, page_fill=fill)


def test_scale_and_large_scores(ctx):
    b = workload.paged_batch([700, 64], 32, 8)
    q, pool = _make(b, 5)
    q = (q.float() * 8).to(torch.bfloat16)  # scores ~ O(10^2): max-shift stability
    out, lse, _ = _run(ctx, b, q, pool, scale=0.5)
    _check(b, q, pool, out, lse, scale=0.5)


def test_repeat_launch_counters_rearmed(ctx):
    # The in-kernel merge ticket is reset by the last arriver; repeated launches
    # (and graph replays) must give identical results.
    rng = np.random.default_rng(9)
    b = workload.paged_batch(rng.integers(500, 5000, size=16).tolist(), 32, 8, frame_order="shuffled")
    q, pool = _make(b, 6)
    out1, lse1, att = _run(ctx, b, q, pool)
    for _ in range(3):
        att.launch()
    torch.cuda.synchronize()
    out2 = att._keep[6].cpu().double().numpy()
    lse2 = att._keep[7].cpu().double().numpy()
    assert np.array_equal(out1, out2) and np.array_equal(lse1, lse2)


def test_lse_merge_identity(ctx):
    # A request computed whole equals the lse_merge (attn_merge.hpp:86-100) of
    # the same request split into two shards at a page boundary.
    L = 3000
    whole = workload.paged_batch([L], 32, 8)
    q, pool = _make(whole, 8)
    o_w, l_w, _ = _run(ctx, whole, q, pool)
    split = workload.PagedBatch(np.array([1600, L - 1600], np.int64), np.array([0, 100, 188], np.int32),
                                whole.block_table.copy(), whole.num_frames, 32, 8)
    q2 = q.expand(2, -1, -1).contiguous()
    o_s, l_s, _ = _run(ctx, split, q2, pool)
    m = np.maximum(l_s[0], l_s[1])
    w0, w1 = np.exp(l_s[0] - m), np.exp(l_s[1] - m)
    merged = (w0[:, None] * o_s[0] + w1[:, None] * o_s[1]) / (w0 + w1)[:, None]
    lse_m = m + np.log(w0 + w1)
    assert np.abs(merged - o_w[0]).max() < 1e-4
    assert np.abs(lse_m - l_w[0]).max() < 1e-4


@pytest.mark.parametrize("frame_order", ["lifo", "shuffled"])
def test_cfg2_full_size_all_shards(ctx, frame_order):
    """BASELINE configs[1] at full size on bench.py's own inputs (64 requests, 1K-32K, 32q/8kv,
    1,068,741 tokens): every shard and head against the fp64 oracle, for the bench's LIFO
    frames and for shuffled frames; plus shard-order invariance over the whole batch."""
    from paper_2605_21100_b200.attention import DecodeAttention
    dev = torch.device("cuda:0")
    b, pool, q = workload.cfg2_bench_inputs(dev, frame_order=frame_order)
    att = DecodeAttention(ctx, 32, 8, max_shards=64)
    out, lse = att(q, pool, torch.from_numpy(b.block_table).to(dev), torch.from_numpy(b.cu_pages).to(dev),
                   torch.from_numpy(b.shard_len).to(dev))
    torch.cuda.synchronize()
    o = out.cpu().double().numpy()
    l = lse.cpu().double().numpy()
    rel, dl = _check(b, q.cpu(), pool.cpu(), o, l)
    print(f"cfg2 {frame_order}: 64 shards x 32 heads, worst O rel-L2 {rel:.3e}, LSE |d| {dl:.3e}")
    # reversed shard order -> different CTA cut points, same answers (split invariance)
    rev = list(range(63, -1, -1))
    sl2 = b.shard_len[rev]
    cu2 = np.concatenate([[0], np.cumsum((sl2 + 15) // 16)]).astype(np.int32)
    bt2 = np.concatenate([b.block_table[b.cu_pages[r]:b.cu_pages[r + 1]] for r in rev]).astype(np.int32)
    att2 = DecodeAttention(ctx, 32, 8, max_shards=64)
    out2, lse2 = att2(q[rev].contiguous(), pool, torch.from_numpy(bt2).to(dev), torch.from_numpy(cu2).to(dev),
                      torch.from_numpy(sl2).to(dev))
    torch.cuda.synchronize()
    o1 = o[rev]
    o2 = out2.cpu().double().numpy()
    relr = np.linalg.norm(o1 - o2, axis=-1) / np.linalg.norm(o1, axis=-1)
    # P is rounded to bf16 relative to the running max, which depends on the cut points:
    # ~2^-9 relative differences are expected (each run is within the 2e-2 oracle bound).
    assert relr.max() < 1e-2, relr.max()
    assert np.abs(l[rev] - lse2.cpu().double().numpy()).max() < 1e-4


# ---- K1-f32: the fp32 production precision (rel <= 1e-5) --------------------------
F32_TOL = 1e-5


def _run_f32(ctx, batch, q, pool, page_fill=None):
    from paper_2605_21100_b200.attention import DecodeAttention
    dev = torch.device("cuda:0")
    att = DecodeAttention(ctx, batch.num_q_heads, batch.num_kv_heads, batch.head_dim, batch.page_size,
                          max_shards=max(len(batch.shard_len), 1), dtype="f32")
    pf = torch.from_numpy(page_fill).to(dev) if page_fill is not None else None
    out, lse = att(q.to(dev), pool.to(dev), torch.from_numpy(batch.block_table).to(dev),
                   torch.from_numpy(batch.cu_pages).to(dev), torch.from_numpy(batch.shard_len).to(dev),
                   page_fill=pf)
    torch.cuda.synchronize()
    o, l = out.cpu().double().numpy(), lse.cpu().double().numpy()
    ro, rl = oracle_lib.paged_decode_f32in_f64(batch, q.numpy(), pool.numpy(), page_fill)
    ne = batch.shard_len > 0
    assert np.all(np.isneginf(l[~ne])) and np.all(o[~ne] == 0)
    rel = (np.linalg.norm(o[ne] - ro[ne], axis=-1) / np.linalg.norm(ro[ne], axis=-1)).max() if ne.any() else 0.0
    dl = np.abs(l[ne] - rl[ne]) / np.maximum(1.0, np.abs(rl[ne])) if ne.any() else np.zeros(1)
    assert rel <= F32_TOL, f"fp32 O rel-L2 {rel:.3e}"
    assert dl.max() <= F32_TOL, f"fp32 LSE {dl.max():.3e}"
    return rel, dl.max()


@pytest.mark.parametrize("hq,hkv,page", [(8, 8, 16), (32, 8, 16), (16, 4, 16), (8, 1, 16), (8, 8, 12), (8, 8, 64)])
def test_f32_paged_matches_oracle(ctx, hq, hkv, page):
    rng = np.random.default_rng(hq * 7 + hkv + page)
    lens = [1, 7, page, page + 1, 0, 333, 2500] + rng.integers(1, 4096, size=9).tolist()
    b = workload.paged_batch(lens, hq, hkv, 128, page, frame_order="shuffled", seed=5, spare_frames=17)
    g = torch.Generator().manual_seed(hq + hkv)
    q = torch.randn(len(lens), hq, 128, generator=g)
    pool = torch.randn(b.num_frames, 2, hkv, page, 128, generator=g)
    rel, dl = _run_f32(ctx, b, q, pool)
    print(f"f32 hq={hq} hkv={hkv} page={page}: rel {rel:.2e} lse {dl:.2e}")


def test_f32_page_fill_and_large_scores(ctx):
    lens = [46, 300, 77, 5000]
    b = workload.paged_batch(lens, 8, 8, frame_order="shuffled", seed=4, spare_frames=5)
    fill = np.full(int(b.cu_pages[-1]), 16, np.uint8)
    for r, L in enumerate(lens):
        fill[b.cu_pages[r + 1] - 1] = L - 16 * (b.cu_pages[r + 1] - b.cu_pages[r] - 1)
    fill[1] = 14
    fill[b.cu_pages[1] + 3] = 9
    fill[b.cu_pages[3] + 100] = 2
    g = torch.Generator().manual_seed(3)
    q = torch.randn(4, 8, 128, generator=g) * 6      # scores O(10^2)
    pool = torch.randn(b.num_frames, 2, 8, 16, 128, generator=g)
    _run_f32(ctx, b, q, pool, page_fill=fill)
