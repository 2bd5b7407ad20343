"""Seeded synthetic inputs for the BASELINE configs.

Lengths use the reference's portable RNG: std::mt19937_64 (standard-specified
output) with `uniform01` / `uniform_int` of workload.hpp:18-26, so the same
seed gives the same request lengths as the reference (cfg2: seed 0, 64
requests in [1024, 32768], sum 1,068,741).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_M64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (w=64, n=312, m=156, r=31)."""

    def __init__(self, seed: int):
        mt = [0] * 312
        mt[0] = seed & _M64
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self.mt, self.i = mt, 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            y = x >> 1
            if x & 1:
                y ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ y
        self.i = 0

    def __call__(self) -> int:
        if self.i >= 312:
            self._twist()
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M64


def uniform01(rng: MT19937_64) -> float:  # workload.hpp:19-21
    return float(rng() >> 11) * (2.0 ** -53)


def uniform_int(rng: MT19937_64, lo: int, hi: int) -> int:  # workload.hpp:22-26
    u = uniform01(rng)
    v = lo + int(u * float(hi - lo + 1))
    return hi if v > hi else v


def lengths(seed: int, n: int, lo: int, hi: int):
    rng = MT19937_64(seed)
    return [uniform_int(rng, lo, hi) for _ in range(n)]


@dataclass
class PagedBatch:
    """Host description of one instance's decode-attention inputs."""
    shard_len: np.ndarray      # int64 [R]
    cu_pages: np.ndarray       # int32 [R+1]
    block_table: np.ndarray    # int32 [P]
    num_frames: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int = 128
    page_size: int = 16

    @property
    def total_tokens(self) -> int:
        return int(self.shard_len.sum())

    def kv_bytes(self) -> int:
        """Algorithmic K+V bytes (token counts, not page-rounded)."""
        return self.total_tokens * self.num_kv_heads * self.head_dim * 2 * 2

    def algorithmic_bytes(self) -> int:
        """SURVEY §8(d) K1 bytes/step: KV + Q(bf16) + O(fp32) + LSE(fp32) + block table."""
        R = len(self.shard_len)
        hq, d = self.num_q_heads, self.head_dim
        return (self.kv_bytes() + R * hq * d * 2 + R * hq * d * 4 + R * hq * 4
                + int(self.cu_pages[-1]) * 4)


def paged_batch(shard_len, num_q_heads, num_kv_heads, head_dim=128, page_size=16,
                frame_order: str = "lifo", seed: int = 0, spare_frames: int = 0) -> PagedBatch:
    """Lay shards out in a paged pool.

    frame_order "lifo": frames handed out in ascending order, exactly as
    make_cluster's LIFO stack + GlobalPageTable::allocate do for a fresh
    instance (page_table.cpp:36-37, 143-145).  "shuffled": a seeded random
    permutation (what a long-running instance looks like after frees).
    """
    shard_len = np.asarray(shard_len, dtype=np.int64)
    pages = (shard_len + page_size - 1) // page_size
    cu = np.zeros(len(shard_len) + 1, dtype=np.int32)
    cu[1:] = np.cumsum(pages)
    P = int(cu[-1])
    nf = P + spare_frames
    if frame_order == "lifo":
        bt = np.arange(P, dtype=np.int32)
    else:
        bt = np.random.default_rng(seed).permutation(nf)[:P].astype(np.int32)
    return PagedBatch(shard_len, cu, bt, max(nf, 1), num_q_heads, num_kv_heads, head_dim, page_size)


def cfg2_lengths():
    """BASELINE configs[1]: 64 requests, uniform_int(mt19937_64(0), 1024, 32768)."""
    return lengths(0, 64, 1024, 32768)


def cfg2_bench_inputs(device, seed: int = 1234, frame_order: str = "lifo"):
    """The cfg2 step bench.py times, as (PagedBatch, pool, q): the 64 cfg2 requests laid out
    with `frame_order`, a bf16 pool and bf16 queries drawn on `device` from a seeded
    generator (pool first, then q).  The parity tests check these exact tensors."""
    import torch
    b = paged_batch(cfg2_lengths(), 32, 8, 128, 16, frame_order=frame_order, seed=seed,
                    spare_frames=0 if frame_order == "lifo" else 4096)
    g = torch.Generator(device=device).manual_seed(seed)
    pool = torch.randn(b.num_frames, 2, 8, 16, 128, generator=g, device=device, dtype=torch.bfloat16)
    q = torch.randn(64, 32, 128, generator=g, device=device, dtype=torch.bfloat16)
    return b, pool, q


# ------------------------------------------------------------------ traces
# Input generation for the trace-driven benches: the reference's Table-1
# distributions and gen_trace (workload.hpp:28-74, workload.cpp:11-106),
# restated so a seed gives the same (arrival, seq_len, output_len) sequence.
SHAREGPT4O = [(1, 1000, 85.7 / 99.9), (1000, 10000, 10.7 / 99.9), (10000, 100000, 3.5 / 99.9)]
GITHUB_ISSUE = [(100000, 500000, 0.6506), (500000, 1000000, 0.3494)]


def sample_length(dist, rng: MT19937_64, log_uniform: bool = False) -> int:  # workload.cpp:56-71
    import math
    u = uniform01(rng)
    cum = 0.0
    lo, hi, _ = dist[-1]
    for b in dist:
        cum += b[2]
        if u < cum:
            lo, hi, _ = b
            break
    if log_uniform:
        a, c = math.log(lo), math.log(hi)
        v = int(math.exp(a + uniform01(rng) * (c - a)))
        return min(max(v, lo), hi - 1)
    return uniform_int(rng, lo, hi - 1)


def gen_trace(seed: int, long_ratio: float, rate_per_s: float, duration_s: float, poisson: bool = False,
              output_len=(64, 512), short=SHAREGPT4O, long=GITHUB_ISSUE):
    """[(id, arrival_ms, seq_len, output_len)], sorted by arrival (workload.cpp:73-106)."""
    import math
    rng = MT19937_64(seed)
    horizon = duration_s * 1000.0
    arrivals = []
    if not poisson:
        gap = 1000.0 / rate_per_s
        i = 0
        while i * gap < horizon:
            arrivals.append(i * gap)
            i += 1
    else:
        t, mean_gap = 0.0, 1000.0 / rate_per_s
        while True:
            t += -math.log(1.0 - uniform01(rng)) * mean_gap
            if t >= horizon:
                break
            arrivals.append(t)
    out = []
    for i, a in enumerate(arrivals):
        is_long = long_ratio > 0.0 and uniform01(rng) < long_ratio
        L = sample_length(long if is_long else short, rng)
        out.append((i, a, L, uniform_int(rng, output_len[0], output_len[1])))
    return out


# ------------------------------------------------------------------ trace files
# The reference's trace file format (workload.hpp:70-72, workload.cpp:108-137):
# header "id,arrival_ms,seq_len,output_len", one request per line, arrival with three
# decimals; loading skips the header and blank lines and orders by (arrival, id).
TRACE_HEADER = "id,arrival_ms,seq_len,output_len"


def write_trace_csv(trace) -> str:
    """trace: [(id, arrival_ms, seq_len, output_len)] -> CSV text (write_trace_csv)."""
    lines = [TRACE_HEADER]
    lines += [f"{int(i)},{a:.3f},{int(L)},{int(o)}" for i, a, L, o in trace]
    return "\n".join(lines) + "\n"


def load_trace_csv(text: str):
    """CSV text -> [(id, arrival_ms, seq_len, output_len)] sorted by (arrival, id) (load_trace_csv).
    An empty file is a ConfigError, as in the reference (workload.cpp:120)."""
    from ._capi import ConfigError
    lines = text.split("\n")
    if text == "":
        raise ConfigError("empty trace file")
    out = []
    for line in lines[1:]:
        if not line:
            continue
        f = line.split(",")
        out.append((int(f[0]), float(f[1]), int(f[2]), int(f[3])))
    out.sort(key=lambda r: (r[1], r[0]))
    return out
