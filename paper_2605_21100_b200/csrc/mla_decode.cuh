// SPDX-License-Identifier: Apache-2.0
//
// K10: MLA-shaped split-KV paged decode attention on tcgen05 (SURVEY §8f #1,
// the DeepSeek-V3 absorbed-latent layout of cfg5).
//
// Semantics, per shard r and q-head h (reference attn_merge.hpp:53-82 applied
// with keys = the 576-wide cache rows and values = their first 512 columns):
//   s_j = scale * <q_h, kv_j[0:576]>
//   O_h = sum_j softmax(s)_j kv_j[0:512]           (normalised, hpp:79)
//   lse = max_j s_j + ln sum_j exp(s_j - max)      (natural log, hpp:80)
// Stream-K partials merge as lse_merge (hpp:86-100).
//
// Design (B200):
//   * 128 heads x 576 / 512 at bf16 is ~242 flop per cache byte: at the ridge
//     of B200 (HBM ~6.5 TB/s vs ~1.6 PF dense bf16), so the products run on
//     tcgen05 with fp32 accumulators in TMEM.
//   * O (128 x 512 fp32) alone is a whole SM's TMEM, so a CTA pair
//     (cluster of 2, cta_group::2, M = 128) shares every MMA: CTA c owns heads
//     [64c, 64c+64) and half of each B operand; its TMEM holds its 64 rows
//     folded into 128 lanes (lanes 64.. carry the second half of N).  Per CTA:
//     S split over K into S_A + S_B (two MMA chains), each double-buffered,
//     4 x 64 columns; O 256 columns.
//   * A tile is 128 tokens of one shard.  S = Q K^T: N = 128 tokens, CTA c
//     streams tokens [64c, 64c+64) x 576 (9 K boxes of 64).  O += P V: N = 256
//     latent dims per MMA, CTA c streams dims [256j+128c, +128) of all 128
//     tokens (MN-major B straight from the cache rows; the re-read hits L2).
//   * Warps: 4 softmax warps per CTA (thread t <-> TMEM lane t); 4 MMA warps in
//     the leader, one per accumulator chain (S_A, S_B, O's two latent halves);
//     2 TMA issuer warps per ring (QA: K boxes 0-4, QB: 5-8 from HBM; V0, V1 from
//     L2), 2-CTA TMA completing on the leader's barriers.  Shared memory: Q 72
//     KB, one P buffer (16 KB), 17 ring stages of 8 KB (5 + 4 + 4 + 4).  The
//     softmax keeps a per-row reference max and rescales O in TMEM only when
//     the max grows by more than 2^8.
//   * Persistent pairs, stream-K over tiles: every pair streams the same number
//     of tiles whatever the 1K..512K length skew; cut shards leave partials in
//     a per-pair slot and a third, fully parallel launch merges them.  Tile
//     scan -> decode -> merge are PDL-chained.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

#include "exchange.cuh"
#include "ptx.cuh"
#include "tc05.cuh"

namespace dcp {
namespace mla {

constexpr int H = 128;               // q heads (64 per CTA of the pair)
constexpr int DL = 512;              // latent width = V width
constexpr int DR = 64;               // rope width
constexpr int DK = DL + DR;          // 576 = K width
constexpr int NKB = DK / 64;         // 9 K boxes of 64 columns
constexpr int TILE = 128;            // tokens per pair tile
constexpr int HT = TILE / 2;         // tokens per CTA in S = Q K^T
constexpr int STAGE = 8192;          // ring stage bytes
constexpr int Q_BYTES = NKB * 8192;  // 64 heads x 576 bf16 per CTA
constexpr int P_BYTES = 2 * 8192;    // 64 heads x 128 tokens bf16 per CTA
#ifndef MLA_NP
#define MLA_NP 1
#endif
// P buffers (softmax -> PV).  One buffer frees 16 KB for a fourth stage on each PV ring: the
// L2-fed PV rings were the ones starving (0.381 -> 0.364 ms cfg2-shaped; P x3 with 2 + 2 PV stages:
// 0.51 ms; QB below 4 stages: 0.41-0.54 ms; profiles/r2_k10_ab.md)
constexpr int NP = MLA_NP;
// Four accumulator chains, each issued by its own MMA warp and fed by its own ring: an
// accumulating 2-CTA M=128 MMA costs ~120 ns whatever its N, but chains issued by different
// warps overlap (tools/probe/mma_rate.cu).  S = Q K^T is split over K into two accumulators
// (boxes 0-4 -> S_A, 5-8 -> S_B; the softmax adds them), O += P V over the two latent halves.
enum Ring { RQA = 0, RQB = 1, RV0 = 2, RV1 = 3, NRING = 4 };
constexpr int QA_BOXES = 5;          // K boxes [0, 5) -> S_A, [5, 9) -> S_B ...
constexpr int QB_SHARE = 2;          // ... except box 4's last 2 k-steps, issued by the S_B chain: 18 + 18 MMAs
#ifndef MLA_RS_QA
#define MLA_RS_QA 5
#define MLA_RS_QB 4
#define MLA_RS_V0 4
#define MLA_RS_V1 4
#endif
__host__ __device__ constexpr int ring_stages(int k) {
    return k == RQA ? MLA_RS_QA : k == RQB ? MLA_RS_QB : k == RV0 ? MLA_RS_V0 : MLA_RS_V1;
}
__host__ __device__ constexpr int ring_first(int k) { return k == 0 ? 0 : ring_first(k - 1) + ring_stages(k - 1); }
// The S_B chain reads box 4 from the QA ring's stage 4, which therefore always holds box 4.
static_assert(MLA_RS_QA == QA_BOXES, "the QA ring has one stage per QA box");
constexpr int NSTAGES = ring_first(NRING);  // 15 stages of 8 KB
constexpr int OFF_Q = 0;
constexpr int OFF_P = OFF_Q + Q_BYTES;
constexpr int OFF_RING = OFF_P + NP * P_BYTES;
constexpr int OFF_MISC = OFF_RING + NSTAGES * STAGE;
// misc: barriers then exchange scratch.  Ring "full" barriers live in the leader: 1 arrival
// (the leader's issuer, expecting both CTAs' bytes) + tx; "empty" in each CTA: 1 (MMA commit multicast).
constexpr int BAR_FULL = 0;                        // [NSTAGES]
constexpr int BAR_EMPTY = BAR_FULL + 8 * NSTAGES;  // [NSTAGES]
constexpr int BAR_QFULL = BAR_EMPTY + 8 * NSTAGES; // leader: 1 + tx
constexpr int BAR_QEMPTY = BAR_QFULL + 8;     // each: 2 (both QK MMA warps)
constexpr int BAR_SFULL = BAR_QEMPTY + 8;     // [2 S buffers][A, B] each: 1
constexpr int BAR_SEMPTY = BAR_SFULL + 32;    // [2] leader: 8 softmax warps
constexpr int BAR_PFULL = BAR_SEMPTY + 16;    // [NP] leader: 8
constexpr int BAR_PEMPTY = BAR_PFULL + 8 * NP;  // [NP] each: 2 (both PV MMA warps)
constexpr int BAR_OEMPTY = BAR_PEMPTY + 8 * NP; // leader: 8
constexpr int TMEM_SLOT = BAR_OEMPTY + 8;
constexpr int RED = 512;                      // float[2][128] exchange scratch
constexpr int MISC_BYTES = RED + 2 * 128 * 4;
constexpr int SMEM = 1024 + OFF_MISC + MISC_BYTES;
// Warp roles: 0-3 softmax (thread t <-> TMEM lane t), 4-7 MMA issuers of rings QA/QB/V0/V1
// (leader CTA), 8-11 TMA issuers of the same rings (both CTAs; the lanes of a warp issue the
// boxes of a stage together, since one thread issues a box only every ~200 cycles,
// tools/probe/tma_bw.cu).
constexpr int W_MMA = 4;
constexpr int W_TMA = 8;
#ifndef MLA_NTW
#define MLA_NTW 2
#endif
constexpr int NTW = MLA_NTW;                  // TMA issuer warps per ring
constexpr int THREADS = 32 * (W_TMA + NTW * NRING);
constexpr uint32_t TM_SA = 0;                 // S_A buffers: cols [0,64), [64,128)
constexpr uint32_t TM_SB = 128;               // S_B buffers: cols [128,192), [192,256)
constexpr uint32_t TM_O = 256;                // O: chunk j at 256 + 128 j
constexpr float RESCALE_LOG2 = 8.f;           // rescale O only when the max grows by > 2^8

static_assert(SMEM <= 232448, "shared memory");

struct MlaParams {
    const int32_t* block_table;  // [P] frame ids
    const int32_t* cu_pages;     // [R+1]
    const int64_t* shard_len;    // [R]
    const uint8_t* page_fill;    // [P] or nullptr
    const int32_t* cu_tiles;     // [R+1] (workspace, from mla_tile_scan_kernel)
    int32_t* pair_t0;            // [pairs+1] first tile of each pair (workspace, from mla_tile_scan_kernel)
    int32_t num_pairs;
    int32_t seg_tiles;           // stream-K weight of a shard start, in tiles (pipeline drain + Q load + O epilogue)
    float* out;                  // [R][128][512]
    float* lse;                  // [R][128]
    float* ws_acc;               // [2*pairs][128][512]
    float* ws_ml;                // [2*pairs][128][2]
    int32_t num_shards;
    int32_t num_frames;
    float scale_log2;
    int32_t dbg;                 // bottleneck experiments (compile-time -DDCP_MLA_DBG=n only): 1 = no MMAs, 2 = no softmax math
    long long* trace;            // optional [256][8] globaltimer stamps of pair 0 + [256][3] per pair (dcp_mla_set_trace)
    // ---- routed mode (DCP exchange, exchange.cuh); NULL for a local call.  Q rows come from
    // this instance's receive pool (the q map spans both parities: row (parity * q_rows + r) * H),
    // each shard's Q-route flag is awaited before its Q load, and O / LSE go to m_r's result
    // slot, whose flag the merge launch publishes once every write of the shard is done.
    const XchgPeers* xp;
    const int32_t* n_mrow;       // [R] row of the shard's request in m_r's M list
    const int32_t* n_moe;        // [R] m_r
    const int32_t* num_shards_ptr;  // device-resident R (overrides num_shards)
    int32_t* tickets;            // [n_max] merge-CTA tickets per shard (self-resetting)
    int32_t q_rows;              // rows of one parity of the receive pool (n_max)
};

__device__ __forceinline__ int num_shards_of(const MlaParams& p) {
    return p.num_shards_ptr ? *p.num_shards_ptr : p.num_shards;
}
__device__ __forceinline__ uint32_t epoch_of(const MlaParams& p) { return p.xp ? *p.xp->epoch : 0u; }
// shard r's normalised output row block [H][DL] and LSE [H]: local, or m_r's result slot
__device__ __forceinline__ float* out_of(const MlaParams& p, int r, uint32_t ep) {
    if (!p.xp) return p.out + static_cast<size_t>(r) * H * DL;
    const XchgPeers& x = *p.xp;
    return xres_o(x, p.n_moe[r], ep) + (static_cast<size_t>(p.n_mrow[r]) * x.W + x.self) * H * DL;
}
__device__ __forceinline__ float* lse_of(const MlaParams& p, int r, uint32_t ep) {
    if (!p.xp) return p.lse + static_cast<size_t>(r) * H;
    const XchgPeers& x = *p.xp;
    return xres_lse(x, p.n_moe[r], ep) + (static_cast<size_t>(p.n_mrow[r]) * x.W + x.self) * H;
}

__device__ __forceinline__ long long gtime() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// trace slot k of pair-0 tile g (one writer per slot)
#define MLA_TRACE(g, k)                                                                     \
    do {                                                                                    \
        if (p.trace && pair == 0 && (g) < 256) p.trace[(g) * 8 + (k)] = gtime();            \
    } while (0)

// Weighted stream-K: pair k streams tiles [pair_t0[k], pair_t0[k+1]).  The split is even in
// work = tiles + seg_tiles per shard, because every shard a pair starts costs it a pipeline
// drain, a Q load and an O epilogue (at equal tile counts, pairs with 2-3 segments were the
// slowest: profiles/r1_k10_trace_pairs.txt).  seg_tiles = 4 (env DCP_MLA_SEG_TILES) measured
// best: long mix 0.327 -> 0.309 ms, cfg2-shaped unchanged (its spread is mostly SM speed).
__device__ __forceinline__ int pair_of_tile(const int32_t* pair_t0, int np, int t) {
    int lo = 0, hi = np - 1;  // last pair k with pair_t0[k] <= t (the non-empty one holding t)
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pair_t0[mid] <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}
__device__ __forceinline__ bool pair_nonempty(const int32_t* pair_t0, int k) { return pair_t0[k] < pair_t0[k + 1]; }

// cu_tiles[r] = sum_{s<r} ceil(pages_s / pages_per_tile).
template <int PAGE>
__global__ void __launch_bounds__(1024) mla_tile_scan_kernel(MlaParams p) {
    pdl_trigger();  // the decode launch's prologue may overlap this scan
    constexpr int PPT = TILE / PAGE;
    __shared__ int32_t warp_sum[32];
    __shared__ int32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int R = num_shards_of(p);
    for (int base = 0; base < R; base += 1024) {
        const int r = base + threadIdx.x;
        int v = 0;
        if (r < R) v = (p.cu_pages[r + 1] - p.cu_pages[r] + PPT - 1) / PPT;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31) >= o) x += y;
        }
        if ((threadIdx.x & 31) == 31) warp_sum[threadIdx.x >> 5] = x;
        __syncthreads();
        if (threadIdx.x < 32) {
            int w = warp_sum[threadIdx.x];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, w, o);
                if (threadIdx.x >= o) w += y;
            }
            warp_sum[threadIdx.x] = w;
        }
        __syncthreads();
        const int excl = carry + x - v + ((threadIdx.x >> 5) ? warp_sum[(threadIdx.x >> 5) - 1] : 0);
        if (r < R) const_cast<int32_t*>(p.cu_tiles)[r] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) const_cast<int32_t*>(p.cu_tiles)[R] = carry;
    __syncthreads();
    // pair_t0[k]: the tile at work unit floor(k W / NP), W = T + seg_tiles R, shard r spanning
    // work [cu_tiles[r] + seg_tiles r, +seg_tiles + tiles_r) with its start cost first
    const int64_t T = carry, X = p.seg_tiles, NP = p.num_pairs;
    const int64_t Wt = T + X * R;
    for (int k = threadIdx.x; k <= NP; k += blockDim.x) {
        const int64_t U = k * Wt / NP;
        int t;
        if (k == NP) {
            t = static_cast<int>(T);
        } else {
            int lo = 0, hi = R;  // last r with cu_work[r] <= U
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (p.cu_tiles[mid] + X * mid <= U) lo = mid; else hi = mid - 1;
            }
            const int64_t off = U - (p.cu_tiles[lo] + X * lo);
            t = lo >= R ? static_cast<int>(T) : p.cu_tiles[lo] + static_cast<int>(off > X ? off - X : 0);
        }
        p.pair_t0[k] = t;
    }
}

// Segment walk shared by every role: the pair's tile range [t_begin, t_end)
// cut at shard boundaries.
struct SegWalk {
    int t, t_end, r;
    __device__ __forceinline__ SegWalk(const int32_t* cu_tiles, int R, int t_begin, int t_end_)
        : t(t_begin), t_end(t_end_) {
        int lo = 0, hi = R - 1;  // last r with cu_tiles[r] <= t_begin
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (cu_tiles[mid] <= t_begin) lo = mid; else hi = mid - 1;
        }
        r = lo;
    }
};

template <int PAGE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    mla_decode_kernel(const __grid_constant__ CUtensorMap q_map, const __grid_constant__ CUtensorMap kvq_map,
                      const __grid_constant__ CUtensorMap kvp_map, const MlaParams p) {
    constexpr int PPT = TILE / PAGE;  // pages per tile
    constexpr int BQ = PAGE < HT ? PAGE : HT;  // rows per TMA box, QK stages (kvq_map)
    constexpr int BP = PAGE < 32 ? PAGE : 32;  // rows per TMA box, PV stages (kvp_map)
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t misc = sbase + OFF_MISC;
    const uint32_t cta = tc::cluster_ctarank();
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.x >> 1;
    // PDL-launched after the tile scan: the merge launch may queue now; this grid's prologue
    // (barriers, TMEM, cluster sync) overlaps the scan, which it waits for before reading its
    // tile ranges (griddepcontrol is a no-op for a plain launch)
    pdl_trigger();

    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGES; ++s) {
            mbar_init(misc + BAR_FULL + 8 * s, 1);
            // QA stage 4 (box 4) is released by both QK chains
            mbar_init(misc + BAR_EMPTY + 8 * s, s == ring_first(RQA) + QA_BOXES - 1 ? 2 : 1);
        }
        mbar_init(misc + BAR_QFULL, 1);
        mbar_init(misc + BAR_QEMPTY, 2);
        for (int b = 0; b < 2; ++b) {
            mbar_init(misc + BAR_SFULL + 16 * b, 1);
            mbar_init(misc + BAR_SFULL + 16 * b + 8, 1);
            mbar_init(misc + BAR_SEMPTY + 8 * b, 8);
        }
        for (int b = 0; b < NP; ++b) {
            mbar_init(misc + BAR_PFULL + 8 * b, 8);
            mbar_init(misc + BAR_PEMPTY + 8 * b, 2);
        }
        mbar_init(misc + BAR_OEMPTY, 8);
        fence_mbar_init();
    }
    if (warp == W_TMA && lane == 0) {
        tma_prefetch_desc(&q_map);
        tma_prefetch_desc(&kvq_map);
        tma_prefetch_desc(&kvp_map);
    }
    if (warp == 0) tc::tmem_alloc<2>(misc + TMEM_SLOT, 512);
    tc::fence_before_sync();
    tc::cluster_sync();
    tc::fence_after_sync();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + OFF_MISC + TMEM_SLOT);
    const uint32_t lead = tc::mapa(misc, 0);  // leader's misc block (shared::cluster)
    pdl_wait();
    const int R = num_shards_of(p);
    const uint32_t ep = epoch_of(p);
    const int t_begin = p.pair_t0[pair];
    const int t_end = p.pair_t0[pair + 1];
    // trace tail (dcp_mla_set_trace): per pair start, end and SM at [2048 + 3 pair + 0..2]
    if (p.trace && cta == 0 && threadIdx.x == 0 && pair < 256) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.trace[2048 + 3 * pair] = gtime();
        p.trace[2048 + 3 * pair + 2] = smid;
    }

    if (t_begin < t_end) {
        if (warp >= W_TMA) {
            // ===================== TMA issuers (both CTAs, one warp per ring) =====================
            // Ring k streams its stages in tile order; lane 0 waits for the slot and (leader)
            // posts both CTAs' bytes, then lanes 0..n-1 issue the stage's n boxes together.
            // Frame ids: lane i holds page i of the tile, prefetched a tile ahead.
            const int rk = (warp - W_TMA) / NTW, ik = (warp - W_TMA) % NTW;  // ring, issuer within it
            const int nst = ring_stages(rk), s0 = ring_first(rk);
            const uint32_t ring = sbase + OFF_RING + s0 * STAGE;
            const int bi = ik + NTW * lane;  // the box of a stage this lane issues
            const uint64_t pol_first = l2_policy_evict_first();
            const uint64_t pol_norm = tc::l2_policy_evict_normal();
            uint32_t it = 0;
            int seg = 0;
            auto stage_begin = [&]() {
                const uint32_t s = it % nst;
                if (lane == 0) {
                    tc::mbar_wait_sleep(misc + BAR_EMPTY + 8 * (s0 + s), ((it / nst) & 1) ^ 1);
                    if (cta == 0 && ik == 0) mbar_arrive_expect_tx(misc + BAR_FULL + 8 * (s0 + s), 2 * STAGE);
                }
                __syncwarp();
                ++it;
                return s;
            };
            SegWalk w(p.cu_tiles, R, t_begin, t_end);
            while (w.t < w.t_end) {
                while (p.cu_tiles[w.r + 1] <= w.t) ++w.r;
                const int r = w.r;
                const int t0 = w.t, t1 = min(p.cu_tiles[r + 1], w.t_end);
                const int pg_begin = p.cu_pages[r], pg_end = p.cu_pages[r + 1];
                const int r_first_tile = p.cu_tiles[r];
                // pages past the shard get an out-of-bounds frame -> TMA zero fill
                auto tile_frame = [&](int t) {
                    const int pg = pg_begin + (t - r_first_tile) * PPT + lane;
                    return (lane < PPT && pg < pg_end) ? __ldg(p.block_table + pg) : p.num_frames;
                };
                int f_cur = tile_frame(t0);
                if (rk == RQA && ik == 0) {  // Q rows of this shard (this CTA's 64 heads), 9 boxes issued by lanes 0-8
                    if (lane == 0) {
                        if (seg > 0) tc::mbar_wait_sleep(misc + BAR_QEMPTY, (seg - 1) & 1);
                        if (p.xp) {  // routed: the Q-route put of this row must have landed
                            wait_flag(xq_flag(*p.xp, p.xp->self, ep) + r, ep, p.xp->wc,
                                      (SITE_K10_Q << 24) | (r & 0xffff));
                            asm volatile("fence.proxy.async.global;" ::: "memory");  // generic -> TMA reads
                        }
                        if (cta == 0) mbar_arrive_expect_tx(misc + BAR_QFULL, 2 * Q_BYTES);
                    }
                    __syncwarp();
                    const int qrow = p.xp ? (static_cast<int>(ep & 1) * p.q_rows + r) * H : r * H;
                    if (lane < NKB)
                        tc::tma_load_2d_pair(sbase + OFF_Q + lane * 8192, &q_map, 64 * lane,
                                             qrow + 64 * static_cast<int>(cta), lead + BAR_QFULL, pol_norm);
                }
                for (int t = t0; t < t1; ++t) {
                    const int f_next = (t + 1 < t1) ? tile_frame(t + 1) : 0;
                    if (rk == RQA || rk == RQB) {
                        // QK stage b: this CTA's HT tokens x K box b, as boxes of BQ = min(PAGE, HT) rows
                        const int b_lo = rk == RQA ? 0 : QA_BOXES, b_hi = rk == RQA ? QA_BOXES : NKB;
                        for (int b = b_lo; b < b_hi; ++b) {
                            const uint32_t s = stage_begin();
                            const int u = HT * static_cast<int>(cta) + bi * BQ;  // this lane's box
                            const int f = __shfl_sync(0xffffffffu, f_cur, (u / PAGE) & 31);
                            if (bi < HT / BQ)
                                tc::tma_load_3d_pair(ring + s * STAGE + bi * BQ * 128, &kvq_map, 64 * b, u % PAGE, f,
                                                     lead + BAR_FULL + 8 * (s0 + s), pol_norm);
                        }
                    } else {
                        // PV stage q of latent half j: tokens [32q, 32q+32) x dims [256j + 128c, +128),
                        // 2 column boxes of 64 x (32 / BP) row boxes of BP = min(PAGE, 32)
                        const int j = rk - RV0;
                        for (int q = 0; q < TILE / 32; ++q) {
                            const uint32_t s = stage_begin();
                            const int k = bi >> 1, bx = bi & 1;
                            const int u = 32 * q + k * BP;
                            const int f = __shfl_sync(0xffffffffu, f_cur, (u / PAGE) & 31);
                            if (bi < 2 * (32 / BP))
                                tc::tma_load_3d_pair(ring + s * STAGE + bx * 4096 + k * BP * 128, &kvp_map,
                                                     64 * (4 * j + 2 * static_cast<int>(cta) + bx), u % PAGE, f,
                                                     lead + BAR_FULL + 8 * (s0 + s), pol_first);
                        }
                    }
                    f_cur = f_next;
                }
                ++seg;
                w.t = t1;
                ++w.r;
            }
        } else if (warp >= W_MMA) {
            // ===================== MMA issuers (leader CTA, whole warp; one elected lane issues) ======
            // Warp W_MMA + k drains ring k: QA / QB accumulate S_A / S_B, V0 / V1 the two latent
            // halves of O.  Ring waits are polled by lane 0 and the slot re-broadcast, so every
            // value feeding a tcgen05.mma stays warp-uniform.
            if (cta == 0) {
                const int rk = warp - W_MMA;
                const int nst = ring_stages(rk), s0 = ring_first(rk);
                constexpr uint32_t ID_QK = tc::idesc_bf16_f32(128, 128, false, false);
                constexpr uint32_t ID_PV = tc::idesc_bf16_f32(128, 256, false, true);
                uint32_t it = 0;
                uint32_t g = 0;  // pair tile counter (S / P buffers)
                int seg = 0;
                long long wait_ns = 0, n_wait = 0, n_ready = 0;  // diagnostics (trace rows 252-255)
                const long long t_mma0 = gtime();
                auto wait_full = [&]() -> uint32_t {
                    const uint32_t s = it % nst;
                    if (lane == 0) {
                        const uint32_t bar = misc + BAR_FULL + 8 * (s0 + s), par = (it / nst) & 1;
                        if (p.trace) {
                            if (mbar_try_wait(bar, par)) {
                                ++n_ready;
                            } else {
                                const long long a0 = gtime();
                                mbar_wait(bar, par);
                                wait_ns += gtime() - a0;
                                ++n_wait;
                            }
                        } else {
                            mbar_wait(bar, par);
                        }
                    }
                    __syncwarp();
                    tc::fence_after_sync();
                    ++it;
                    return __shfl_sync(0xffffffffu, s, 0);
                };
                // base descriptors; the 14-bit start-address field never carries (smem < 256 KB)
                const uint64_t dQ = tc::sdesc_sw128(sbase + OFF_Q, 16, 1024);
                const uint64_t dR = tc::sdesc_sw128(sbase + OFF_RING + s0 * STAGE, 16, 1024);
                const uint64_t dRA = tc::sdesc_sw128(sbase + OFF_RING + ring_first(RQA) * STAGE, 16, 1024);
                const uint64_t dRV = tc::sdesc_sw128(sbase + OFF_RING + s0 * STAGE, 4096, 1024);
                const uint64_t dP = tc::sdesc_sw128(sbase + OFF_P, 16, 1024);
                const bool is_qk = rk == RQA || rk == RQB;
                SegWalk w(p.cu_tiles, R, t_begin, t_end);
                while (w.t < w.t_end) {
                    while (p.cu_tiles[w.r + 1] <= w.t) ++w.r;
                    const int t0 = w.t, t1 = min(p.cu_tiles[w.r + 1], w.t_end);
                    if (is_qk) {
                        tc::mbar_wait_sleep(misc + BAR_QFULL, seg & 1);
                        tc::fence_after_sync();
                    }
                    for (int t = t0; t < t1; ++t, ++g) {
                        const uint32_t sb = g & 1;
                        if (is_qk) {
                            // ---- S_A / S_B [sb] = Q K^T over this chain's K boxes ----
                            if (lane == 0 && rk == RQA) MLA_TRACE(g, 0);
                            if (g >= 2) tc::mbar_wait_sleep(misc + BAR_SEMPTY + 8 * sb, ((g >> 1) + 1) & 1);
                            tc::fence_after_sync();
                            const int b_lo = rk == RQA ? 0 : QA_BOXES, b_hi = rk == RQA ? QA_BOXES : NKB;
                            const uint32_t dst = tmem + (rk == RQA ? TM_SA : TM_SB) + 64 * sb;
                            constexpr int SB4 = QA_BOXES - 1;  // the shared box / QA stage
                            if (rk == RQB) {  // S_B starts with box 4's last QB_SHARE k-steps
                                if (lane == 0) mbar_wait(misc + BAR_FULL + 8 * (ring_first(RQA) + SB4), g & 1);
                                __syncwarp();
                                tc::fence_after_sync();
                                const uint64_t a0 = dQ + ((SB4 * 8192) >> 4), b0 = dRA + ((SB4 * STAGE) >> 4);
#pragma unroll
                                for (int kk = 4 - QB_SHARE; kk < 4; ++kk)
                                    if (!(p.dbg & 1))
                                        tc::mma2_bf16_ss_warp(dst, a0 + 2 * kk, b0 + 2 * kk, ID_QK, kk != 4 - QB_SHARE);
                                tc::commit2_mc_warp(misc + BAR_EMPTY + 8 * (ring_first(RQA) + SB4), 0x3);
                            }
                            for (int b = b_lo; b < b_hi; ++b) {
                                const uint32_t s = wait_full();
                                const uint64_t a0 = dQ + ((b * 8192) >> 4), b0 = dR + ((s * STAGE) >> 4);
                                const int kk_hi = b == SB4 ? 4 - QB_SHARE : 4;
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk)
                                    if (kk < kk_hi && !(p.dbg & 1))
                                        tc::mma2_bf16_ss_warp(dst, a0 + 2 * kk, b0 + 2 * kk, ID_QK,
                                                              rk == RQB || ((b - b_lo) | kk) != 0);
                                tc::commit2_mc_warp(misc + BAR_EMPTY + 8 * (s0 + s), 0x3);
                            }
                            tc::commit2_mc_warp(misc + BAR_SFULL + 16 * sb + 8 * rk, 0x3);
                            if (lane == 0 && rk == RQA) MLA_TRACE(g, 1);
                            if (t == t1 - 1) tc::commit2_mc_warp(misc + BAR_QEMPTY, 0x3);
                        } else {
                            // ---- O[j] += P[sb] V[j] over 4 token quarters ----
                            const int j = rk - RV0;
                            const bool first = t == t0;
                            const uint32_t pb = g % NP;
                            tc::mbar_wait_sleep(misc + BAR_PFULL + 8 * pb, (g / NP) & 1);
                            if (first && seg > 0) tc::mbar_wait_sleep(misc + BAR_OEMPTY, (seg - 1) & 1);
                            tc::fence_after_sync();
                            if (lane == 0 && rk == RV0) MLA_TRACE(g, 2);
                            const uint64_t pd = dP + ((pb * P_BYTES) >> 4);
                            for (int q = 0; q < TILE / 32; ++q) {
                                const uint32_t s = wait_full();
                                const uint64_t b0 = dRV + ((s * STAGE) >> 4);
#pragma unroll
                                for (int kk = 0; kk < 2; ++kk) {
                                    const int ks = 2 * q + kk;  // 16-token k-step of the tile
                                    const uint64_t ad = pd + (((ks >> 2) * 8192 + (ks & 3) * 32) >> 4);
                                    if (!(p.dbg & 1))
                                        tc::mma2_bf16_ss_warp(tmem + TM_O + 128 * j, ad, b0 + ((kk * 2048) >> 4), ID_PV,
                                                              !(first && ks == 0));
                                }
                                tc::commit2_mc_warp(misc + BAR_EMPTY + 8 * (s0 + s), 0x3);
                            }
                            tc::commit2_mc_warp(misc + BAR_PEMPTY + 8 * pb, 0x3);
                            if (lane == 0 && rk == RV0) MLA_TRACE(g, 3);
                        }
                    }
                    ++seg;
                    w.t = t1;
                    ++w.r;
                }
                if (p.trace && pair == 0 && lane == 0) {
                    const int row = 252 + rk;
                    p.trace[row * 8 + 0] = gtime() - t_mma0;
                    p.trace[row * 8 + 1] = wait_ns;
                    p.trace[row * 8 + 2] = n_wait;
                    p.trace[row * 8 + 3] = n_ready;
                }
            }
        } else if (warp < 4) {
            // ===================== softmax / correction / epilogue (warps 0-3, both CTAs) ==========
            const int tid = threadIdx.x;        // == TMEM lane
            const int hl = tid & 63;            // head within this CTA
            const int half = tid >> 6;          // token half of S / dim half of O
            const int head = 64 * static_cast<int>(cta) + hl;
            const uint32_t tl = tmem + (static_cast<uint32_t>(warp * 32) << 16);
            float* red = reinterpret_cast<float*>(smem + OFF_MISC + RED);
            const int partner = tid ^ 64;
            uint32_t g = 0;
            int seg = 0;
            SegWalk w(p.cu_tiles, R, t_begin, t_end);
            while (w.t < w.t_end) {
                while (p.cu_tiles[w.r + 1] <= w.t) ++w.r;
                const int r = w.r;
                const int t0 = w.t, t1 = min(p.cu_tiles[r + 1], w.t_end);
                const int r_first = p.cu_tiles[r], r_last = p.cu_tiles[r + 1];
                const int pg_begin = p.cu_pages[r], pg_end = p.cu_pages[r + 1];
                const int64_t len = p.shard_len[r];
                float m_used = -INFINITY, l_run = 0.f;
                for (int t = t0; t < t1; ++t, ++g) {
                    const uint32_t sb = g & 1;
                    // valid tokens of this thread's 4 chunks
                    int nvalid[4];
                    {
                        const int ti = t - r_first;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int chunk = 4 * half + k;
                            const int pi = ti * PPT + (chunk * 16) / PAGE;  // page index within the shard
                            const int off = (chunk * 16) % PAGE;
                            int fill = 0;
                            if (pg_begin + pi < pg_end) {
                                if (p.page_fill) fill = p.page_fill[pg_begin + pi];
                                else {
                                    const int64_t rem = len - static_cast<int64_t>(pi) * PAGE;
                                    fill = rem < PAGE ? static_cast<int>(rem) : PAGE;
                                }
                            }
                            nvalid[k] = min(16, max(0, fill - off));
                        }
                    }
                    tc::mbar_wait_sleep(sbase + OFF_MISC + BAR_SFULL + 16 * sb, (g >> 1) & 1);
                    tc::mbar_wait_sleep(sbase + OFF_MISC + BAR_SFULL + 16 * sb + 8, (g >> 1) & 1);
                    tc::fence_after_sync();
                    if (tid == 0 && cta == 0) MLA_TRACE(g, 4);
                    if (p.dbg & 2) {  // experiment: pass S / P through without the softmax math
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive_cluster(lead + BAR_SEMPTY + 8 * sb);
                        if (g >= NP) tc::mbar_wait_sleep(sbase + OFF_MISC + BAR_PEMPTY + 8 * (g % NP), ((g / NP) + 1) & 1);
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive_cluster(lead + BAR_PFULL + 8 * (g % NP));
                        m_used = 0.f;
                        l_run = 1.f;
                        continue;
                    }
                    float s[64];
                    float mx = -INFINITY;
#pragma unroll
                    for (int c = 0; c < 2; ++c) {  // S = S_A + S_B, 32 columns at a time
                        uint32_t va[32], vb[32];
                        tc::tmem_ld32(tl + TM_SA + 64 * sb + 32 * c, va);
                        tc::tmem_ld32(tl + TM_SB + 64 * sb + 32 * c, vb);
                        tc::tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const int j = 32 * c + i;
                            const bool ok = (j & 15) < nvalid[j >> 4];
                            s[j] = ok ? (__uint_as_float(va[i]) + __uint_as_float(vb[i])) * p.scale_log2 : -INFINITY;
                            mx = fmaxf(mx, s[j]);
                        }
                    }
                    tc::fence_before_sync();
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive_cluster(lead + BAR_SEMPTY + 8 * sb);
                    red[tid] = mx;
                    named_bar_sync(1, 128);
                    mx = fmaxf(mx, red[partner]);
                    named_bar_sync(1, 128);  // red reusable
                    if (tid == 0 && cta == 0) MLA_TRACE(g, 6);
                    bool rescale = false;
                    float alpha = 1.f;
                    if (t == t0) {
                        m_used = mx;
                    } else if (mx > m_used + RESCALE_LOG2) {
                        alpha = fast_exp2(m_used - mx);
                        m_used = mx;
                        rescale = true;
                    }
                    float ps = 0.f;
#pragma unroll
                    for (int j = 0; j < 64; ++j) {
                        s[j] = fast_exp2(s[j] - m_used);
                        ps += s[j];
                    }
                    l_run = l_run * alpha + ps;
                    // P buffer g % NP is free once PV(g - NP) completed
                    const uint32_t pb = g % NP;
                    if (g >= NP) tc::mbar_wait_sleep(sbase + OFF_MISC + BAR_PEMPTY + 8 * pb, ((g / NP) + 1) & 1);
                    if (tid == 0 && cta == 0) MLA_TRACE(g, 7);
                    {
                        uint8_t* prow = smem + OFF_P + pb * P_BYTES + half * 8192 + hl * 128;
#pragma unroll
                        for (int ch = 0; ch < 8; ++ch) {
                            uint4 v;
                            v.x = pack_bf16x2(s[8 * ch + 0], s[8 * ch + 1]);
                            v.y = pack_bf16x2(s[8 * ch + 2], s[8 * ch + 3]);
                            v.z = pack_bf16x2(s[8 * ch + 4], s[8 * ch + 5]);
                            v.w = pack_bf16x2(s[8 * ch + 6], s[8 * ch + 7]);
                            *reinterpret_cast<uint4*>(prow + ((ch ^ (hl & 7)) << 4)) = v;
                        }
                    }
                    // O *= alpha once PV(g-1) has landed.  tcgen05.ld/st are warp-collective, so the
                    // whole warp waits and rewrites its lanes if any lane needs it (alpha = 1 elsewhere).
                    if (__any_sync(0xffffffffu, rescale)) {
                        tc::mbar_wait_sleep(sbase + OFF_MISC + BAR_PEMPTY + 8 * ((g - 1) % NP), ((g - 1) / NP) & 1);
                        tc::fence_after_sync();
                        for (int c = 0; c < 256; c += 32) {
                            uint32_t ov[32];
                            tc::tmem_ld32(tl + TM_O + c, ov);
                            tc::tmem_wait_ld();
#pragma unroll
                            for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * alpha);
                            tc::tmem_st32(tl + TM_O + c, ov);
                        }
                        tc::tmem_wait_st();
                    }
                    tc::fence_proxy_async_smem();
                    tc::fence_before_sync();
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive_cluster(lead + BAR_PFULL + 8 * pb);
                    if (tid == 0 && cta == 0) MLA_TRACE(g, 5);
                }
                // ---- epilogue of segment [t0, t1) of shard r ----
                tc::mbar_wait_sleep(sbase + OFF_MISC + BAR_PEMPTY + 8 * ((g - 1) % NP), ((g - 1) / NP) & 1);
                tc::fence_after_sync();
                red[tid] = l_run;
                named_bar_sync(1, 128);
                const float l_tot = l_run + red[partner];
                named_bar_sync(1, 128);
                const bool complete = (t0 == r_first) && (t1 == r_last);
                const int slot = 2 * pair + (t0 == t_begin ? 0 : 1);
                const float inv = complete ? 1.f / l_tot : 1.f;
                float* dst = complete ? out_of(p, r, ep) + static_cast<size_t>(head) * DL
                                      : p.ws_acc + (static_cast<size_t>(slot) * H + head) * DL;
#pragma unroll 1
                for (int c = 0; c < 256; c += 32) {
                    uint32_t ov[32];
                    tc::tmem_ld32(tl + TM_O + c, ov);
                    tc::tmem_wait_ld();
                    const int j = c >> 7, x0 = c & 127;
                    float4* d4 = reinterpret_cast<float4*>(dst + 256 * j + 128 * half + x0);
#pragma unroll
                    for (int v = 0; v < 8; ++v)
                        d4[v] = make_float4(__uint_as_float(ov[4 * v]) * inv, __uint_as_float(ov[4 * v + 1]) * inv,
                                            __uint_as_float(ov[4 * v + 2]) * inv, __uint_as_float(ov[4 * v + 3]) * inv);
                }
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive_cluster(lead + BAR_OEMPTY);
                if (complete) {
                    if (half == 0) lse_of(p, r, ep)[head] = (m_used + __log2f(l_tot)) * 0.69314718055994530942f;
                } else if (half == 0) {  // cut segment: (max, sum) of the partial; mla_merge_kernel combines
                    __stcg(reinterpret_cast<float2*>(p.ws_ml) + (static_cast<size_t>(slot) * H + head),
                           make_float2(m_used, l_tot));
                }
                ++seg;
                w.t = t1;
                ++w.r;
            }
        }
    }

    tc::fence_before_sync();
    tc::cluster_sync();
    if (p.trace && cta == 0 && threadIdx.x == 0 && pair < 256) p.trace[2048 + 3 * pair + 1] = gtime();
    if (warp == 0) tc::tmem_dealloc<2>(tmem, 512);
}

// Stream-K combine (lse_merge, attn_merge.hpp:86-100, in the log2 domain): every shard cut
// by a pair-range boundary has one partial per pair that touched it.  One CTA per
// (shard, 16-head group, column quarter), one warp per head.  A shard cut over at most
// MERGE_SHORT pairs (the common case: a boundary or two) is merged whole by its quarter-0 CTA,
// all 512 columns per warp; a longer one (a 512K request spans ~50 pairs) spreads its columns
// over four CTAs, so 32 SMs share it.  Uncut shards exit at once; zero-token shards write
// O = 0, LSE = -inf.  A separate launch keeps long shards off any one pair's tail.
constexpr int MERGE_QUARTERS = 4;
constexpr int MERGE_SHORT = 8;
// One warp merges head qh's columns [4*col4, +4*32*NV) over slots a..b.  Slot weights live in
// lanes (32 slots per chunk, read once) and are broadcast by shuffle, so the main loop only
// streams the partial rows: U slots x NV float4 per lane in flight.
template <int NV, int U>
__device__ __forceinline__ void merge_cols(const MlaParams& p, int a, int b, int r_first, int r, int qh, int col4,
                                          float mmax, bool write_lse) {
    auto slot_of = [&](int k) { return (k == a && r_first != p.pair_t0[k]) ? 2 * k + 1 : 2 * k; };
    const int lane = threadIdx.x & 31;
    float den = 0.f;
    float4 num[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) num[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c0 = a; c0 <= b; c0 += 32) {
        const int kl = c0 + lane;
        float w = 0.f;
        int sl_l = slot_of(a);
        if (kl <= b && pair_nonempty(p.pair_t0, kl)) {
            sl_l = slot_of(kl);
            const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.ws_ml) + (static_cast<size_t>(sl_l) * H + qh));
            w = fast_exp2(ml.x - mmax);
            den += w * ml.y;
        }
        const int n = min(32, b - c0 + 1);
        for (int j0 = 0; j0 < n; j0 += U) {
            float wj[U];
            float4 x[U][NV];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = (j0 + u) & 31;  // lanes past n hold w = 0 and a valid slot
                wj[u] = __shfl_sync(0xffffffffu, w, j);
                if (j0 + u >= 32) wj[u] = 0.f;  // the last round of a full chunk wraps
                const int sl = __shfl_sync(0xffffffffu, sl_l, j);
                const float4* src =
                    reinterpret_cast<const float4*>(p.ws_acc + (static_cast<size_t>(sl) * H + qh) * DL) + col4;
#pragma unroll
                for (int v = 0; v < NV; ++v) x[u][v] = __ldcg(src + lane + 32 * v);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    num[v].x += wj[u] * x[u][v].x;
                    num[v].y += wj[u] * x[u][v].y;
                    num[v].z += wj[u] * x[u][v].z;
                    num[v].w += wj[u] * x[u][v].w;
                }
        }
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) den += __shfl_xor_sync(0xffffffffu, den, s);
    const float dinv = 1.f / den;
    const uint32_t ep = epoch_of(p);
    float4* o = reinterpret_cast<float4*>(out_of(p, r, ep) + static_cast<size_t>(qh) * DL) + col4;
#pragma unroll
    for (int v = 0; v < NV; ++v)
        o[lane + 32 * v] = make_float4(num[v].x * dinv, num[v].y * dinv, num[v].z * dinv, num[v].w * dinv);
    if (write_lse && lane == 0) lse_of(p, r, ep)[qh] = (mmax + __log2f(den)) * 0.69314718055994530942f;
}

// Routed mode: the last of the shard's CTAs publishes its Res-route flag.  Every CTA fences
// at system scope before its ticket, so the release covers all of the shard's remote writes,
// including those of the decode launch (complete shards), which finished before this launch.
__device__ __forceinline__ void merge_done(const MlaParams& p, int r) {
    if (!p.xp) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const int n = gridDim.y * gridDim.z;
        if (atomicAdd(p.tickets + r, 1) == n - 1) {
            p.tickets[r] = 0;
            const XchgPeers& x = *p.xp;
            const uint32_t ep = *x.epoch;
            st_release_sys(xres_flag(x, p.n_moe[r], ep) + static_cast<size_t>(p.n_mrow[r]) * x.W + x.self, ep);
        }
    }
}

__global__ void __launch_bounds__(512, 2) mla_merge_kernel(MlaParams p, int num_pairs) {
    pdl_trigger();
    pdl_wait();  // PDL-launched after the decode grid: its partials
    const int r = blockIdx.x;
    if (r >= num_shards_of(p)) return;  // routed launches cover n_max shards
    const int r_first = p.cu_tiles[r], r_last = p.cu_tiles[r + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qh = blockIdx.y * 16 + warp;
    constexpr int QV = DL / 4 / MERGE_QUARTERS;  // float4 columns per quarter (32)
    const uint32_t ep = epoch_of(p);
    if (r_first == r_last) {  // zero-token shard: O = 0, LSE = -inf (its merge weight is 0)
        reinterpret_cast<float4*>(out_of(p, r, ep) + static_cast<size_t>(qh) * DL)[blockIdx.z * QV + lane] =
            make_float4(0.f, 0.f, 0.f, 0.f);
        if (blockIdx.z == 0 && lane == 0) lse_of(p, r, ep)[qh] = -INFINITY;
        merge_done(p, r);
        return;
    }
    const int a = pair_of_tile(p.pair_t0, num_pairs, r_first);
    const int b = pair_of_tile(p.pair_t0, num_pairs, r_last - 1);
    const bool short_span = b - a < MERGE_SHORT;
    // a == b: one pair covered the whole shard and wrote the final output
    if (a != b && (!short_span || blockIdx.z == 0)) {
        auto slot_of = [&](int k) { return (k == a && r_first != p.pair_t0[k]) ? 2 * k + 1 : 2 * k; };
        float mmax = -INFINITY;
        for (int k = a + lane; k <= b; k += 32) {
            if (!pair_nonempty(p.pair_t0, k)) continue;
            mmax = fmaxf(mmax, __ldcg(p.ws_ml + (static_cast<size_t>(slot_of(k)) * H + qh) * 2));
        }
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) mmax = fmaxf(mmax, __shfl_xor_sync(0xffffffffu, mmax, s));
        if (short_span)
            merge_cols<MERGE_QUARTERS, 2>(p, a, b, r_first, r, qh, 0, mmax, true);
        else
            merge_cols<1, 6>(p, a, b, r_first, r, qh, blockIdx.z * QV, mmax, blockIdx.z == 0);
    }
    merge_done(p, r);
}

}  // namespace mla
}  // namespace dcp
