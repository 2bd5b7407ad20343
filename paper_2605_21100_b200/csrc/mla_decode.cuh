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
//     S double-buffered 2 x 64 columns, O 256 columns.
//   * A tile is 128 tokens of one shard.  S = Q K^T: N = 128 tokens, CTA c
//     streams tokens [64c, 64c+64) x 576 (9 K boxes of 64).  O += P V: N = 256
//     latent dims per MMA, CTA c streams dims [256j+128c, +128) of all 128
//     tokens (MN-major B straight from the cache rows; the re-read hits L2).
//   * One producer warp per CTA (TMA, 2-CTA form: completion bytes land on the
//     leader's barrier), one MMA thread in the leader, four softmax warps per
//     CTA (thread t <-> TMEM lane t).  The softmax keeps a per-row reference
//     max and rescales O in TMEM only when the max grows by more than 2^8.
//   * Persistent pairs, stream-K over tiles: every pair streams the same number
//     of tiles whatever the 1K..512K length skew; cut shards leave partials in
//     a per-pair slot, the last pair to finish a shard merges (device ticket).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

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
constexpr int CHUNKS = TILE / 16;    // 16-token TMA chunks per tile
constexpr int STAGE = 8192;          // ring stage bytes
constexpr int NS = 15;               // ring stages
constexpr int Q_BYTES = NKB * 8192;  // 64 heads x 576 bf16 per CTA
constexpr int P_BYTES = 2 * 8192;    // 64 heads x 128 tokens bf16 per CTA
constexpr int OFF_Q = 0;
constexpr int OFF_P = OFF_Q + Q_BYTES;
constexpr int OFF_RING = OFF_P + 2 * P_BYTES;
constexpr int OFF_MISC = OFF_RING + NS * STAGE;
// misc: barriers then exchange scratch
constexpr int BAR_FULL = 0;             // [NS] leader: 2 producer arrivals + tx
constexpr int BAR_EMPTY = BAR_FULL + 8 * NS;  // [NS] each CTA: 1 (MMA commit multicast)
constexpr int BAR_QFULL = BAR_EMPTY + 8 * NS; // leader: 2 + tx
constexpr int BAR_QEMPTY = BAR_QFULL + 8;     // each: 1
constexpr int BAR_SFULL = BAR_QEMPTY + 8;     // [2] each: 1
constexpr int BAR_SEMPTY = BAR_SFULL + 16;    // [2] leader: 8 softmax warps
constexpr int BAR_PFULL = BAR_SEMPTY + 16;    // [2] leader: 8
constexpr int BAR_PEMPTY = BAR_PFULL + 16;    // [2] each: 1
constexpr int BAR_OEMPTY = BAR_PEMPTY + 16;   // leader: 8
constexpr int TMEM_SLOT = BAR_OEMPTY + 8;
constexpr int LAST_FLAG = TMEM_SLOT + 4;
constexpr int RED = 512;                      // float[2][128] exchange scratch
constexpr int MISC_BYTES = RED + 2 * 128 * 4;
constexpr int SMEM = 1024 + OFF_MISC + MISC_BYTES;
constexpr int THREADS = 192;                  // warps 0-3 softmax, 4 producer, 5 MMA
constexpr uint32_t TM_S = 0;                  // S buffers: cols [0,64), [64,128)
constexpr uint32_t TM_O = 256;                // O: chunk j at 256 + 128 j
constexpr float RESCALE_LOG2 = 8.f;           // rescale O only when the max grows by > 2^8

static_assert(SMEM <= 232448, "shared memory");

struct MlaParams {
    const int32_t* block_table;  // [P] frame ids
    const int32_t* cu_pages;     // [R+1]
    const int64_t* shard_len;    // [R]
    const uint8_t* page_fill;    // [P] or nullptr
    const int32_t* cu_tiles;     // [R+1] (workspace, from mla_tile_scan_kernel)
    float* out;                  // [R][128][512]
    float* lse;                  // [R][128]
    float* ws_acc;               // [2*pairs][128][512]
    float* ws_ml;                // [2*pairs][128][2]
    int32_t* counters;           // [2R]
    int32_t num_shards;
    int32_t num_frames;
    float scale_log2;
};

__device__ __forceinline__ int pair_of_tile(int64_t t, int64_t T, int64_t np) {
    return static_cast<int>(((t + 1) * np + T - 1) / T - 1);
}
__device__ __forceinline__ bool pair_nonempty(int64_t k, int64_t T, int64_t np) {
    return T >= np || (k * T / np) < ((k + 1) * T / np);
}

// cu_tiles[r] = sum_{s<r} ceil(pages_s / pages_per_tile); zero-token shards get O = 0, LSE = -inf.
template <int PAGE>
__global__ void __launch_bounds__(1024) mla_tile_scan_kernel(MlaParams p) {
    constexpr int PPT = TILE / PAGE;
    __shared__ int32_t warp_sum[32];
    __shared__ int32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int R = p.num_shards;
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
    // zero-token shards
    for (int r = 0; r < R; ++r) {
        if (p.cu_pages[r + 1] != p.cu_pages[r]) continue;
        float4* o = reinterpret_cast<float4*>(p.out + static_cast<size_t>(r) * H * DL);
        for (int i = threadIdx.x; i < H * DL / 4; i += 1024) o[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (threadIdx.x < H) p.lse[static_cast<size_t>(r) * H + threadIdx.x] = -INFINITY;
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
    mla_decode_kernel(const __grid_constant__ CUtensorMap q_map, const __grid_constant__ CUtensorMap kv_map,
                      const MlaParams p) {
    constexpr int PPT = TILE / PAGE;  // pages per tile
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t misc = sbase + OFF_MISC;
    const uint32_t cta = tc::cluster_ctarank();
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int R = p.num_shards;
    const int64_t T = p.cu_tiles[R];
    const int64_t NP = gridDim.x >> 1;
    const int pair = blockIdx.x >> 1;
    const int t_begin = static_cast<int>(pair * T / NP);
    const int t_end = static_cast<int>((pair + 1) * T / NP);

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(misc + BAR_FULL + 8 * s, 2);
            mbar_init(misc + BAR_EMPTY + 8 * s, 1);
        }
        mbar_init(misc + BAR_QFULL, 2);
        mbar_init(misc + BAR_QEMPTY, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(misc + BAR_SFULL + 8 * b, 1);
            mbar_init(misc + BAR_SEMPTY + 8 * b, 8);
            mbar_init(misc + BAR_PFULL + 8 * b, 8);
            mbar_init(misc + BAR_PEMPTY + 8 * b, 1);
        }
        mbar_init(misc + BAR_OEMPTY, 8);
        fence_mbar_init();
    }
    if (warp == 4 && lane == 0) {
        tma_prefetch_desc(&q_map);
        tma_prefetch_desc(&kv_map);
    }
    if (warp == 0) tc::tmem_alloc<2>(misc + TMEM_SLOT, 512);
    tc::fence_before_sync();
    tc::cluster_sync();
    tc::fence_after_sync();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + OFF_MISC + TMEM_SLOT);
    const uint32_t lead = tc::mapa(misc, 0);  // leader's misc block (shared::cluster)

    if (t_begin < t_end) {
        if (warp == 4) {
            // ===================== TMA producer (both CTAs) =====================
            const uint64_t pol_first = l2_policy_evict_first();
            const uint64_t pol_norm = tc::l2_policy_evict_normal();
            uint32_t it = 0;  // ring counter
            int seg = 0;
            auto stage_begin = [&](uint32_t& dst) {
                const uint32_t s = it % NS;
                if (lane == 0) {
                    mbar_wait(misc + BAR_EMPTY + 8 * s, ((it / NS) & 1) ^ 1);
                    tc::mbar_arrive_expect_tx_cluster(lead + BAR_FULL + 8 * s, STAGE);
                }
                dst = sbase + OFF_RING + s * STAGE;
                return lead + BAR_FULL + 8 * s;
            };
            // QK stage b of a tile: this CTA's 64 tokens (chunks 4c..4c+3) x K box b
            auto qk_stage = [&](int b, int frame_lane) {
                uint32_t dst;
                const uint32_t bar = stage_begin(dst);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int chunk = 4 * cta + k;
                    const int f = __shfl_sync(0xffffffffu, frame_lane, (chunk * 16) / PAGE);
                    if (lane == 0)
                        tc::tma_load_3d_pair(dst + k * 2048, &kv_map, 64 * b, (chunk * 16) % PAGE, f, bar, pol_norm);
                }
                ++it;
            };
            // PV stage (j, q): tokens [32q, 32q+32) x dims [256j + 128c, +128) as 2 boxes of 64
            auto pv_stage = [&](int j, int q, int frame_lane) {
                uint32_t dst;
                const uint32_t bar = stage_begin(dst);
#pragma unroll
                for (int pg = 0; pg < 2; ++pg) {
                    const int chunk = 2 * q + pg;
                    const int f = __shfl_sync(0xffffffffu, frame_lane, (chunk * 16) / PAGE);
#pragma unroll
                    for (int bx = 0; bx < 2; ++bx)
                        if (lane == 0)
                            tc::tma_load_3d_pair(dst + bx * 4096 + pg * 2048, &kv_map,
                                                 64 * (4 * j + 2 * static_cast<int>(cta) + bx), (chunk * 16) % PAGE, f,
                                                 bar, pol_first);
                }
                ++it;
            };
            SegWalk w(p.cu_tiles, R, t_begin, t_end);
            while (w.t < w.t_end) {
                while (p.cu_tiles[w.r + 1] <= w.t) ++w.r;
                const int r = w.r;
                const int t0 = w.t, t1 = min(p.cu_tiles[r + 1], w.t_end);
                const int pg_begin = p.cu_pages[r], pg_end = p.cu_pages[r + 1];
                // Q rows of this shard (this CTA's 64 heads)
                if (lane == 0) {
                    if (seg > 0) mbar_wait(misc + BAR_QEMPTY, (seg - 1) & 1);
                    tc::mbar_arrive_expect_tx_cluster(lead + BAR_QFULL, Q_BYTES);
                    for (int b = 0; b < NKB; ++b)
                        tc::tma_load_2d_pair(sbase + OFF_Q + b * 8192, &q_map, 64 * b, r * H + 64 * static_cast<int>(cta),
                                             lead + BAR_QFULL, pol_norm);
                }
                __syncwarp();
                int prev_frames = 0;
                for (int t = t0; t < t1; ++t) {
                    const int pg0 = pg_begin + (t - p.cu_tiles[r]) * PPT;
                    int frames = p.num_frames;  // out of bounds -> TMA zero fill
                    if (lane < PPT && pg0 + lane < pg_end) frames = __ldg(p.block_table + pg0 + lane);
                    for (int b = 0; b < NKB; ++b) qk_stage(b, frames);
                    if (t > t0)
                        for (int j = 0; j < 2; ++j)
                            for (int q = 0; q < 4; ++q) pv_stage(j, q, prev_frames);
                    prev_frames = frames;
                }
                for (int j = 0; j < 2; ++j)
                    for (int q = 0; q < 4; ++q) pv_stage(j, q, prev_frames);
                ++seg;
                w.t = t1;
                ++w.r;
            }
        } else if (warp == 5) {
            // ===================== MMA issuer (leader CTA, one thread) =====================
            if (cta == 0 && lane == 0) {
                constexpr uint32_t ID_QK = tc::idesc_bf16_f32(128, 128, false, false);
                constexpr uint32_t ID_PV = tc::idesc_bf16_f32(128, 256, false, true);
                uint32_t it = 0;
                uint32_t g = 0;  // pair tile counter (S / P buffers)
                int seg = 0;
                auto wait_full = [&]() -> uint32_t {
                    const uint32_t s = it % NS;
                    tc::mbar_wait_cluster(misc + BAR_FULL + 8 * s, (it / NS) & 1);
                    tc::fence_after_sync();
                    return s;
                };
                auto pv = [&](uint32_t gp, bool first) {
                    const uint32_t pb = gp & 1;
                    tc::mbar_wait_cluster(misc + BAR_PFULL + 8 * pb, (gp >> 1) & 1);
                    if (first && seg > 0) tc::mbar_wait_cluster(misc + BAR_OEMPTY, (seg - 1) & 1);
                    tc::fence_after_sync();
                    const uint32_t pbase = sbase + OFF_P + pb * P_BYTES;
                    for (int j = 0; j < 2; ++j)
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t s = wait_full();
                            const uint32_t st = sbase + OFF_RING + s * STAGE;
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk) {
                                const int ks = 2 * q + kk;  // 16-token k-step of the tile
                                const uint64_t ad = tc::sdesc_sw128(pbase + (ks >> 2) * 8192 + (ks & 3) * 32, 16, 1024);
                                const uint64_t bd = tc::sdesc_sw128(st + kk * 2048, 4096, 1024);
                                tc::mma_bf16_ss<2>(tmem + TM_O + 128 * j, ad, bd, ID_PV, !(first && ks == 0));
                            }
                            tc::commit2_mc(misc + BAR_EMPTY + 8 * s, 0x3);
                            ++it;
                        }
                    tc::commit2_mc(misc + BAR_PEMPTY + 8 * pb, 0x3);
                };
                SegWalk w(p.cu_tiles, R, t_begin, t_end);
                while (w.t < w.t_end) {
                    while (p.cu_tiles[w.r + 1] <= w.t) ++w.r;
                    const int t0 = w.t, t1 = min(p.cu_tiles[w.r + 1], w.t_end);
                    tc::mbar_wait_cluster(misc + BAR_QFULL, seg & 1);
                    tc::fence_after_sync();
                    for (int t = t0; t < t1; ++t, ++g) {
                        const uint32_t sb = g & 1;
                        if (g >= 2) tc::mbar_wait_cluster(misc + BAR_SEMPTY + 8 * sb, ((g >> 1) + 1) & 1);
                        tc::fence_after_sync();
                        for (int b = 0; b < NKB; ++b) {
                            const uint32_t s = wait_full();
                            const uint32_t st = sbase + OFF_RING + s * STAGE;
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                const uint64_t ad = tc::sdesc_sw128(sbase + OFF_Q + b * 8192 + kk * 32, 16, 1024);
                                const uint64_t bd = tc::sdesc_sw128(st + kk * 32, 16, 1024);
                                tc::mma_bf16_ss<2>(tmem + TM_S + 64 * sb, ad, bd, ID_QK, (b | kk) != 0);
                            }
                            tc::commit2_mc(misc + BAR_EMPTY + 8 * s, 0x3);
                            ++it;
                        }
                        tc::commit2_mc(misc + BAR_SFULL + 8 * sb, 0x3);
                        if (t == t1 - 1) tc::commit2_mc(misc + BAR_QEMPTY, 0x3);
                        if (t > t0) pv(g - 1, t - 1 == t0);
                    }
                    pv(g - 1, t1 - 1 == t0);
                    ++seg;
                    w.t = t1;
                    ++w.r;
                }
            }
        } else {
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
                    tc::mbar_wait_cluster(sbase + OFF_MISC + BAR_SFULL + 8 * sb, (g >> 1) & 1);
                    tc::fence_after_sync();
                    uint32_t sv[2][32];
                    tc::tmem_ld32(tl + TM_S + 64 * sb, sv[0]);
                    tc::tmem_ld32(tl + TM_S + 64 * sb + 32, sv[1]);
                    tc::tmem_wait_ld();
                    tc::fence_before_sync();
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive_cluster(lead + BAR_SEMPTY + 8 * sb);
                    float s[64];
                    float mx = -INFINITY;
#pragma unroll
                    for (int j = 0; j < 64; ++j) {
                        const bool ok = (j & 15) < nvalid[j >> 4];
                        s[j] = ok ? __uint_as_float(sv[j >> 5][j & 31]) * p.scale_log2 : -INFINITY;
                        mx = fmaxf(mx, s[j]);
                    }
                    red[tid] = mx;
                    named_bar_sync(1, 128);
                    mx = fmaxf(mx, red[partner]);
                    named_bar_sync(1, 128);  // red reusable
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
                    // P buffer sb is free once PV(g-2) completed
                    if (g >= 2) tc::mbar_wait_cluster(sbase + OFF_MISC + BAR_PEMPTY + 8 * sb, ((g >> 1) + 1) & 1);
                    {
                        uint8_t* prow = smem + OFF_P + sb * P_BYTES + half * 8192 + hl * 128;
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
                        tc::mbar_wait_cluster(sbase + OFF_MISC + BAR_PEMPTY + 8 * ((g - 1) & 1), ((g - 1) >> 1) & 1);
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
                    if (lane == 0) tc::mbar_arrive_cluster(lead + BAR_PFULL + 8 * sb);
                }
                // ---- epilogue of segment [t0, t1) of shard r ----
                tc::mbar_wait_cluster(sbase + OFF_MISC + BAR_PEMPTY + 8 * ((g - 1) & 1), ((g - 1) >> 1) & 1);
                tc::fence_after_sync();
                red[tid] = l_run;
                named_bar_sync(1, 128);
                const float l_tot = l_run + red[partner];
                named_bar_sync(1, 128);
                const bool complete = (t0 == r_first) && (t1 == r_last);
                const int slot = 2 * pair + (t0 == t_begin ? 0 : 1);
                const float inv = complete ? 1.f / l_tot : 1.f;
                float* dst = complete ? p.out + (static_cast<size_t>(r) * H + head) * DL
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
                    if (half == 0) p.lse[static_cast<size_t>(r) * H + head] = (m_used + __log2f(l_tot)) * 0.69314718055994530942f;
                } else {
                    if (half == 0)
                        __stcg(reinterpret_cast<float2*>(p.ws_ml) + (static_cast<size_t>(slot) * H + head),
                               make_float2(m_used, l_tot));
                    __threadfence();
                    named_bar_sync(1, 128);
                    volatile int* last_flag = reinterpret_cast<volatile int*>(smem + OFF_MISC + LAST_FLAG);
                    if (tid == 0) {
                        const int a = pair_of_tile(r_first, T, NP);
                        const int b = pair_of_tile(r_last - 1, T, NP);
                        int nparts = b - a + 1;
                        if (T < NP) {
                            nparts = 0;
                            for (int k = a; k <= b; ++k) nparts += pair_nonempty(k, T, NP);
                        }
                        const int prev = atomicAdd(p.counters + 2 * r + cta, 1);
                        *last_flag = (prev == nparts - 1) ? 1 : 0;
                    }
                    named_bar_sync(1, 128);
                    if (*last_flag) {
                        __threadfence();
                        const int a = pair_of_tile(r_first, T, NP);
                        const int b = pair_of_tile(r_last - 1, T, NP);
                        for (int hh = warp; hh < 64; hh += 4) {
                            const int qh = 64 * static_cast<int>(cta) + hh;
                            float mmax = -INFINITY;
                            for (int k = a; k <= b; ++k) {
                                if (!pair_nonempty(k, T, NP)) continue;
                                const int sl = (k == a && r_first != static_cast<int>(k * T / NP)) ? 2 * k + 1 : 2 * k;
                                mmax = fmaxf(mmax, __ldcg(p.ws_ml + (static_cast<size_t>(sl) * H + qh) * 2));
                            }
                            float den = 0.f;
                            float4 num[4];
#pragma unroll
                            for (int v = 0; v < 4; ++v) num[v] = make_float4(0.f, 0.f, 0.f, 0.f);
                            for (int k = a; k <= b; ++k) {
                                if (!pair_nonempty(k, T, NP)) continue;
                                const int sl = (k == a && r_first != static_cast<int>(k * T / NP)) ? 2 * k + 1 : 2 * k;
                                const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.ws_ml) + (static_cast<size_t>(sl) * H + qh));
                                const float wk = fast_exp2(ml.x - mmax);
                                den += wk * ml.y;
                                const float4* src = reinterpret_cast<const float4*>(p.ws_acc + (static_cast<size_t>(sl) * H + qh) * DL);
#pragma unroll
                                for (int v = 0; v < 4; ++v) {
                                    const float4 x = __ldcg(src + lane + 32 * v);
                                    num[v].x += wk * x.x;
                                    num[v].y += wk * x.y;
                                    num[v].z += wk * x.z;
                                    num[v].w += wk * x.w;
                                }
                            }
                            const float dinv = 1.f / den;
                            float4* o = reinterpret_cast<float4*>(p.out + (static_cast<size_t>(r) * H + qh) * DL);
#pragma unroll
                            for (int v = 0; v < 4; ++v)
                                o[lane + 32 * v] = make_float4(num[v].x * dinv, num[v].y * dinv, num[v].z * dinv, num[v].w * dinv);
                            if (lane == 0) p.lse[static_cast<size_t>(r) * H + qh] = (mmax + __log2f(den)) * 0.69314718055994530942f;
                        }
                        if (tid == 0) p.counters[2 * r + cta] = 0;  // re-arm
                    }
                }
                ++seg;
                w.t = t1;
                ++w.r;
            }
        }
    }

    tc::fence_before_sync();
    tc::cluster_sync();
    if (warp == 0) tc::tmem_dealloc<2>(tmem, 512);
}

}  // namespace mla
}  // namespace dcp
