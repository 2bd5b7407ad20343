// SPDX-License-Identifier: Apache-2.0
//
// K1 + K9: split-KV paged decode attention for sm_100a.
//
// Semantics (per shard r, q-head h):   reference attn_merge.hpp:53-82
//   s_j  = scale * <q, k_j>                      (hpp:66-67)
//   O    = sum_j softmax(s)_j v_j                (hpp:68-79, normalised, hpp:79)
//   lse  = max_j s_j + ln(sum_j exp(s_j - max))  (hpp:80, natural log)
// and the intra-GPU combine of chunk partials follows lse_merge (hpp:86-100):
//   out = sum_k w_k O_k / sum_k w_k,  w_k = exp(lse_k - max lse).
//
// Design (B200):
//   * HBM-bound (GQA-4: ~4 flop/B).  One persistent CTA per SM; the flattened
//     page sequence of all shards is cut into gridDim.x equal page ranges
//     ("stream-K" over pages), so every SM streams the same number of bytes
//     regardless of the 1K..32K length skew.
//   * One producer warp streams whole frames (K and V of every kv-head, the
//     64 KB page of cfg2) into a STAGES-deep shared-memory ring with two 2-D
//     TMA tensor loads per page (128-B swizzle, L2 evict-first), completion
//     tracked by mbarrier transaction counts.
//   * One consumer warp per kv-head: the GQA group's q-heads are the M rows
//     of mma.sync m16n8k16 bf16 tiles (tokens on N for QK^T, head-dim on N for
//     PV), fp32 accumulation, online softmax in the log2 domain.
//   * A shard cut by a range boundary leaves partials (unnormalised O, max,
//     sum) in a per-CTA slot; the last CTA to finish the shard (device-scope
//     atomic ticket) merges them in page order — no second launch.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

#include "exchange.cuh"
#include "ptx.cuh"

namespace dcp {

struct AttnParams {
    const __nv_bfloat16* q;      // [R][HQ][D]
    const int32_t* block_table;  // [P]
    const int32_t* cu_pages;     // [R+1]
    const int64_t* shard_len;    // [R]
    const uint8_t* page_fill;    // [P] or nullptr
    float* out;                  // [R][HQ][D]
    float* lse;                  // [R][HQ]
    float* ws_acc;               // [2*grid][HQ][D]
    float* ws_ml;                // [2*grid][HQ][2]
    int32_t* counters;           // [R]
    int32_t num_shards;
    float scale_log2;            // scale * log2(e)
    // ---- routed mode (DCP exchange, exchange.cuh); all NULL for a local step.  Q and the
    // Q-route flags then come from this instance's receive pool (parity of the epoch).
    const XchgPeers* xp;         // peer pools; outputs go to m_r's result slot
    const int32_t* n_mrow;       // [R] row of the shard's request in m_r's M list
    const int32_t* n_moe;        // [R] m_r
    const int32_t* num_shards_ptr;  // device-resident R (graph replay); overrides num_shards
    const int32_t* total_pages_ptr; // device-resident cu_pages[R] (routed: loaded alongside R)
    long long* trace;            // optional [grid][8] globaltimer stamps per CTA (dcp_k1_set_trace)
    // ---- fused routed step (dcp_decode_step_fused): one launch per step.  FUSE_STEP: this
    // launch is the step's begin_step (fence, epoch e = *epoch + 1, advanced by the CTA whose
    // producer warp takes the grid's ticket last); FUSE_ROUTE: K2's Q-route puts in the prologue; FUSE_MERGE: K3's LSE merges of this
    // instance's M rows in the epilogue (spins on peers' Res-route flags: multi-GPU / W = 1 only).
    uint32_t fuse;
    const void* q_local;         // [m_max][HQ][D] bf16, M-row order (route)
    const int32_t* m_count;      // [W] device M counts (K7)
    const int32_t* m_nrow;       // [M][W] destination rows (route)
    const int32_t* m_k;          // [M] |P_r| (merge)
    const int32_t* m_kv;         // [M][PL_MAXK] P_r in kv_binding order (merge)
    float* mout;                 // [m_max][HQ][D] merged O (merge)
    float* mout_lse;             // [m_max][HQ]
    int32_t* exit_ticket;        // grid exit counter (step)
};
enum : uint32_t { FUSE_STEP = 1, FUSE_ROUTE = 2, FUSE_MERGE = 4 };
#ifndef K9_U
#define K9_U 8  // K9 merge: parts whose partial rows are in flight together (GQA <= 4)
#endif

__device__ __forceinline__ long long k1_gtime() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Fused step, shard r of a request homed here with P_r = {self} (CP 1, m_r = self): its output
// is final — written straight to the merged output, no Res-route slot, flag or merge (the merge
// of a single part is the identity: weight exp(0) = 1, lse unchanged, bit for bit).
template <class P>
__device__ __forceinline__ bool row_final_here(const P& p, int r) {
    return (p.fuse & 4u) && p.n_moe[r] == p.xp->self && p.m_k[p.n_mrow[r]] == 1;
}

// Destination of shard r's normalised partial O / LSE: local [R][HQ][D] for a
// local step, else m_r's result pool slot [mrow][self] (Res-route put, fused).
template <class P>
__device__ __forceinline__ float* row_out(const P& p, int r, int HQ, int D, uint32_t ep) {
    if (!p.xp) return p.out + (size_t)r * HQ * D;
    if (row_final_here(p, r)) return p.mout + (size_t)p.n_mrow[r] * HQ * D;
    const XchgPeers& x = *p.xp;
    return xres_o(x, p.n_moe[r], ep) + ((size_t)p.n_mrow[r] * x.W + x.self) * HQ * D;
}
template <class P>
__device__ __forceinline__ float* row_lse(const P& p, int r, int HQ, uint32_t ep) {
    if (!p.xp) return p.lse + (size_t)r * HQ;
    if (row_final_here(p, r)) return p.mout_lse + (size_t)p.n_mrow[r] * HQ;
    const XchgPeers& x = *p.xp;
    return xres_lse(x, p.n_moe[r], ep) + ((size_t)p.n_mrow[r] * x.W + x.self) * HQ;
}
// Called by thread 0 after a consumer barrier: every warp's stores of row r
// happen-before this system-scope release.
template <class P>
__device__ __forceinline__ void publish_row(const P& p, int r, uint32_t ep) {
    if (row_final_here(p, r)) return;
    const XchgPeers& x = *p.xp;
    st_release_sys(xres_flag(x, p.n_moe[r], ep) + (size_t)p.n_mrow[r] * x.W + x.self, ep);
}

// The same destinations from the shard's routing fields loaded once at the shard's start
// (nm = n_moe[r], nr = n_mrow[r], mk = m_k[nr]): the epilogue / K9 merge after the page loop
// then has no dependent loads on its tail.
struct RowRoute {
    int nm, nr, mk;
};
template <class P>
__device__ __forceinline__ RowRoute row_route(const P& p, int r) {
    RowRoute rr{0, 0, 0};
    if (p.xp) {
        rr.nm = p.n_moe[r];
        rr.nr = p.n_mrow[r];
        if (p.fuse & 4u) rr.mk = p.m_k[rr.nr];
    }
    return rr;
}
template <class P>
__device__ __forceinline__ float* row_out_c(const P& p, int r, const RowRoute& rr, int HQ, int D, uint32_t ep) {
    if (!p.xp) return p.out + (size_t)r * HQ * D;
    const XchgPeers& x = *p.xp;
    if ((p.fuse & 4u) && rr.nm == x.self && rr.mk == 1) return p.mout + (size_t)rr.nr * HQ * D;
    return xres_o(x, rr.nm, ep) + ((size_t)rr.nr * x.W + x.self) * HQ * D;
}
template <class P>
__device__ __forceinline__ float* row_lse_c(const P& p, int r, const RowRoute& rr, int HQ, uint32_t ep) {
    if (!p.xp) return p.lse + (size_t)r * HQ;
    const XchgPeers& x = *p.xp;
    if ((p.fuse & 4u) && rr.nm == x.self && rr.mk == 1) return p.mout_lse + (size_t)rr.nr * HQ;
    return xres_lse(x, rr.nm, ep) + ((size_t)rr.nr * x.W + x.self) * HQ;
}
template <class P>
__device__ __forceinline__ void publish_row_c(const P& p, const RowRoute& rr, uint32_t ep) {
    const XchgPeers& x = *p.xp;
    if ((p.fuse & 4u) && rr.nm == x.self && rr.mk == 1) return;
    st_release_sys(xres_flag(x, rr.nm, ep) + (size_t)rr.nr * x.W + x.self, ep);
}

// SPLIT = false: a ring stage is one whole frame (K and V of every kv-head).
// SPLIT = true:  a ring stage is half a frame (the K part or the V part); the
// K half is released right after QK^T, and the finer ring fits 3.5 frames in
// flight instead of 3 (7 x 32 KB vs 3 x 64 KB at 8 kv-heads).
//
// Pages larger than 16 tokens (page_size 32, 64, ... — ClusterTopology::page_size,
// types.hpp:92) use the split ring with a 3-D tensor map (d, token-in-page,
// frame*2*HKV + kv*HKV + head): each ring item is a 16-token chunk of one
// part of one page, so the consumer code is identical for every page size.
template <int HKV, int G, bool SPLIT = false, int PAGE_ = 16>
struct DecodeCfg {
    static constexpr int D = 128;
    static constexpr int PAGE = PAGE_;
    static constexpr int CHUNKS = PAGE / 16;          // 16-token chunks per page
    static constexpr int HQ = HKV * G;
    static constexpr int ROWS = 2 * HKV * 16;         // 2-D tensor rows per frame (whole-frame ring)
    static constexpr int HALF = HKV * 16;             // rows of one part of one 16-token chunk
    static constexpr int BOX_ROWS = SPLIT ? HALF : ROWS;
    static constexpr int BOX_BYTES = BOX_ROWS * 128;  // one 64-column swizzled box
    static constexpr int STAGE_BYTES = 2 * BOX_BYTES; // a frame, or half a frame when SPLIT
    static constexpr int V_ROW = SPLIT ? 0 : HALF;    // first V row inside a stage
    static constexpr int STAGES_RAW = ((SPLIT ? 224 : 192) * 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_RAW > 16 ? 16 : STAGES_RAW;
    static constexpr int CONSUMERS = HKV;             // warps
    static constexpr int THREADS = (HKV + 1) * 32;
    static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
    static constexpr int SMEM = 1024 + BAR_OFF + 2 * STAGES * 8 + STAGES * 4 + 16;
    static_assert(ROWS <= 256, "TMA box rows");
    static_assert(PAGE % 16 == 0 && (SPLIT || PAGE == 16), "pages > 16 tokens need the split ring");
    static_assert(G <= 16, "group must fit the 16 mma rows");
};

__device__ __forceinline__ int cta_of_page(int64_t p, int64_t P, int64_t grid) {
    // CTA c owns pages [floor(c*P/grid), floor((c+1)*P/grid)).
    return static_cast<int>(udiv64((p + 1) * grid + P - 1, P) - 1);
}
// With fewer pages than CTAs some ranges are empty; those CTAs hold no partial.
__device__ __forceinline__ bool cta_nonempty(int64_t k, int64_t P, int64_t grid) {
    return P >= grid || udiv64(k * P, grid) < udiv64((k + 1) * P, grid);
}

template <int HKV, int G, bool SPLIT = false, int PAGE_ = 16>
__global__ void __launch_bounds__(DecodeCfg<HKV, G, SPLIT, PAGE_>::THREADS, 1)
    splitkv_decode_kernel(const __grid_constant__ CUtensorMap kv_map, const AttnParams p) {
    using C = DecodeCfg<HKV, G, SPLIT, PAGE_>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t smem_base = smem_u32(smem);
    const uint32_t full_bar = smem_base + C::BAR_OFF;
    const uint32_t empty_bar = full_bar + C::STAGES * 8;
    volatile int* last_flag = reinterpret_cast<volatile int*>(smem + C::BAR_OFF + 2 * C::STAGES * 8);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int R = p.num_shards_ptr ? *p.num_shards_ptr : p.num_shards;
    const uint32_t ep = p.xp ? *p.xp->epoch + ((p.fuse & FUSE_STEP) ? 1u : 0u) : 0u;
    const __nv_bfloat16* qbase =
        p.xp ? reinterpret_cast<const __nv_bfloat16*>(xq_recv(*p.xp, p.xp->self, ep)) : p.q;
    const uint32_t* qflag = p.xp ? xq_flag(*p.xp, p.xp->self, ep) : nullptr;
    const int64_t P = p.total_pages_ptr ? *p.total_pages_ptr : p.cu_pages[R];
    const int64_t grid = gridDim.x;
    const int cta = blockIdx.x;
    const int p_begin = static_cast<int>(udiv64(cta * P, grid));
    const int p_end = static_cast<int>(udiv64((cta + 1) * P, grid));

    if (p.trace && threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.trace[cta * 8 + 0] = k1_gtime();
        p.trace[cta * 8 + 6] = smid;
        p.trace[cta * 8 + 7] = p_end - p_begin;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(full_bar + 8 * s, 1);
            mbar_init(empty_bar + 8 * s, C::CONSUMERS);
        }
        fence_mbar_init();
    }
    if (warp == C::CONSUMERS && lane == 0) tma_prefetch_desc(&kv_map);
    __syncthreads();

    if (warp == C::CONSUMERS) {
        // ===================== producer warp =====================
        const uint64_t policy = l2_policy_evict_first();
        for (int base = p_begin; base < p_end; base += 32) {
            const int mine = base + lane;
            int frame = 0;
            if (mine < p_end) frame = __ldg(p.block_table + mine);
            const int n = min(32, p_end - base);
            for (int i = 0; i < n; ++i) {
                const int f = __shfl_sync(0xffffffffu, frame, i);
                if (lane == 0) {
                    const int it = base - p_begin + i;
                    for (int c = 0; c < C::CHUNKS; ++c) {
#pragma unroll
                        for (int part = 0; part < (SPLIT ? 2 : 1); ++part) {
                            const int j = SPLIT ? 2 * (it * C::CHUNKS + c) + part : it;
                            const int s = j % C::STAGES;
                            const uint32_t ph = (j / C::STAGES) & 1;
                            mbar_wait(empty_bar + 8 * s, ph ^ 1);
                            mbar_arrive_expect_tx(full_bar + 8 * s, C::STAGE_BYTES);
                            const uint32_t dst = smem_base + s * C::STAGE_BYTES;
                            if constexpr (SPLIT) {
                                const int z = (f * 2 + part) * HKV;
                                tma_load_3d(dst, &kv_map, 0, c * 16, z, full_bar + 8 * s, policy);
                                tma_load_3d(dst + C::BOX_BYTES, &kv_map, 64, c * 16, z, full_bar + 8 * s, policy);
                            } else {
                                const int row = f * C::ROWS;
                                tma_load_2d(dst, &kv_map, 0, row, full_bar + 8 * s, policy);
                                tma_load_2d(dst + C::BOX_BYTES, &kv_map, 64, row, full_bar + 8 * s, policy);
                            }
                        }
                    }
                }
                __syncwarp();
            }
        }
        if ((p.fuse & FUSE_STEP) && lane == 0) {
            // Fused step: the last CTA to have read the epoch advances it (nothing in this grid
            // reads it again; the next launch reads it after this grid completed).  Taken by the
            // producer once its loads are issued, so the atomic is off the consumers' tail.
            if (atom_add_acq_rel_gpu(p.exit_ticket, 1) == static_cast<int>(gridDim.x) - 1) {
                *p.exit_ticket = 0;
                *p.xp->epoch = ep;
            }
        }
        return;
    }

    // ===================== consumer warps (one per kv-head) =====================
    const int h = warp;
    const int g = lane >> 2;
    const int t = lane & 3;
    constexpr int NCT = C::CONSUMERS * 32;

    if (p.fuse & FUSE_STEP) {
        // begin_step (exchange.cuh): publish done = e-1, wait until every peer is done with e-2,
        // before this CTA's first store into a peer pool (the producer warp only reads KV)
        const XchgPeers& x = *p.xp;
        if (warp == 0) {
            if (cta == 0 && lane == 0) st_relaxed_sys(xdone(x, x.self), ep - 1);
            for (int s = lane; s < x.W; s += 32)
                if (s != x.self) wait_flag(xdone(x, s), ep - 2, x.wc, (SITE_FENCE << 24) | (s << 16), true);
        }
        named_bar_sync(1, NCT);
    }
    if (p.fuse & FUSE_ROUTE) {
        // K2: this CTA's M rows r = cta, cta + grid, ... to every instance of P_r, 16-byte vectors,
        // then a system-scope release of the row's arrival flag (exchange_kernels.cuh protocol)
        const XchgPeers& x = *p.xp;
        const int M = p.m_count[x.self];
        constexpr int VEC = C::HQ * C::D * 2 / 16;
        for (int r = cta; r < M; r += gridDim.x) {
            const uint4* src = reinterpret_cast<const uint4*>(p.q_local) + (size_t)r * VEC;
            for (int s = 0; s < x.W; ++s) {
                const int row = p.m_nrow[(size_t)r * x.W + s];
                if (row < 0 || s == x.self) continue;  // the home's own shard reads Q in place
                uint4* dst = reinterpret_cast<uint4*>(xq_recv(x, s, ep)) + (size_t)row * VEC;
                for (int i = threadIdx.x; i < VEC; i += NCT) dst[i] = __ldg(src + i);
                named_bar_sync(1, NCT);
                if (threadIdx.x == 0) st_release_sys(xq_flag(x, s, ep) + row, ep);
            }
        }
    }

    // Zero-token shards: O = 0, LSE = -inf (weight 0 in any merge).
    for (int r = cta; r < R; r += gridDim.x) {
        if (p.cu_pages[r + 1] == p.cu_pages[r]) {
            float* ob = row_out(p, r, C::HQ, C::D, ep);
            float* lb = row_lse(p, r, C::HQ, ep);
            for (int row = 0; row < G; ++row) {
                float* o = ob + (h * G + row) * C::D;
                reinterpret_cast<float4*>(o)[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (lane == 0) lb[h * G + row] = -INFINITY;
            }
            if (p.xp) {
                named_bar_sync(1, NCT);
                if (threadIdx.x == 0) publish_row(p, r, ep);
            }
        }
    }

    auto attend = [&]() {
    // Per-lane ldmatrix offsets (stage-relative).  Row & 7 == lane & 7 since
    // every head tile starts on an 8-row boundary (128B swizzle atom).
    const int mi = lane >> 3, rr = lane & 7;
    uint32_t k_off[2][4], v_off[8];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int kp = 0; kp < 4; ++kp) {
            const int ks = 2 * kp + (mi >> 1);
            const int box = ks >> 2;
            const int chunk = ((ks & 3) << 1) | (mi & 1);
            const int row = h * 16 + nt * 8 + rr;
            k_off[nt][kp] = box * C::BOX_BYTES + row * 128 + ((chunk ^ rr) << 4);
        }
#pragma unroll
    for (int np = 0; np < 8; ++np) {
        const int tok = (mi & 1) * 8 + rr;
        const int dchunk = 2 * np + (mi >> 1);
        const int box = dchunk >> 3, chunk = dchunk & 7;
        const int row = C::V_ROW + h * 16 + tok;
        v_off[np] = box * C::BOX_BYTES + row * 128 + ((chunk ^ rr) << 4);
    }

    // First shard with a page in [p_begin, ...): last r with cu[r] <= p_begin.
    int r;
    {
        int lo = 0, hi = R;  // answer in [0, R-1]
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (p.cu_pages[mid] <= p_begin) lo = mid; else hi = mid - 1;
        }
        r = lo;
    }

    constexpr bool TWO_HALVES = (G > 8);
    const bool row0_real = g < G;
    const bool row1_real = TWO_HALVES && (g + 8) < G;

    int it = 0;
    int pg = p_begin;
    int fwin = -1, fval = 0;  // page_fill window cache
    while (pg < p_end) {
        while (p.cu_pages[r + 1] <= pg) ++r;  // skip zero-page shards
        const int r_first = p.cu_pages[r];
        const int r_last = p.cu_pages[r + 1];
        const int seg_begin = pg;
        const int seg_end = min(r_last, p_end);
        const int64_t len = p.shard_len[r];

        // Q fragments (A operand, rows = q-heads of this kv group).  Fused step: a request homed
        // here reads its Q row in place (no put to self, no flag).
        const RowRoute rrt = row_route(p, r);
        const bool q_home = (p.fuse & FUSE_ROUTE) && rrt.nm == p.xp->self;
        if (qflag && !q_home) {  // routed: wait for the Q-route put of this row
            if (lane == 0) wait_flag(qflag + r, ep, p.xp->wc, (SITE_K1_Q << 24) | (r & 0xffff));
            __syncwarp();
        }
        uint32_t qa[8][4];
        {
            const __nv_bfloat16* qrow = q_home ? static_cast<const __nv_bfloat16*>(p.q_local) +
                                                     static_cast<size_t>(rrt.nr) * C::HQ * C::D
                                               : qbase + static_cast<size_t>(r) * C::HQ * C::D;
            const __nv_bfloat16* q0 = qrow + (h * G + g) * C::D + 2 * t;
            const __nv_bfloat16* q1 = q0 + 8 * C::D;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                qa[ks][0] = row0_real ? __ldcg(reinterpret_cast<const uint32_t*>(q0 + 16 * ks)) : 0u;
                qa[ks][2] =
                    row0_real ? __ldcg(reinterpret_cast<const uint32_t*>(q0 + 16 * ks + 8)) : 0u;
                qa[ks][1] = row1_real ? __ldcg(reinterpret_cast<const uint32_t*>(q1 + 16 * ks)) : 0u;
                qa[ks][3] =
                    row1_real ? __ldcg(reinterpret_cast<const uint32_t*>(q1 + 16 * ks + 8)) : 0u;
            }
        }

        float acc[16][4];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

        for (; pg < seg_end; ++pg, ++it)
        for (int c = 0; c < C::CHUNKS; ++c) {
            const int jk = SPLIT ? 2 * (it * C::CHUNKS + c) : it;  // ring item of the K part
            const int s = jk % C::STAGES;
            const uint32_t ph = (jk / C::STAGES) & 1;
            const int sv = SPLIT ? (jk + 1) % C::STAGES : s;
            const uint32_t phv = SPLIT ? ((jk + 1) / C::STAGES) & 1 : ph;
            int fill;
            if (p.page_fill) {  // per-page fills, fetched 32 pages per coalesced warp load
                const int w = pg & ~31;
                if (w != fwin) {
                    fwin = w;
                    fval = (w + lane < p_end && w + lane >= p_begin) ? __ldg(p.page_fill + w + lane) : 0;
                }
                fill = __shfl_sync(0xffffffffu, fval, pg - w);
            } else {
                const int64_t rem = len - static_cast<int64_t>(pg - r_first) * C::PAGE;
                fill = rem < C::PAGE ? static_cast<int>(rem) : C::PAGE;
            }
            mbar_wait(full_bar + 8 * s, ph);
            if (p.trace && it == 0 && c == 0 && threadIdx.x == 0) p.trace[cta * 8 + 1] = k1_gtime();
            // valid tokens of this 16-token chunk (chunks past the page's fill are fully masked;
            // chunk 0 always holds >= 1 token, so the running max is finite before any empty chunk)
            fill = min(16, max(0, fill - 16 * c));
            const uint32_t st = smem_base + s * C::STAGE_BYTES;
            const uint32_t stv = smem_base + sv * C::STAGE_BYTES;

            // ---- S = Q K^T (16 rows x 16 tokens) ----
            float sc[2][4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
                for (int kp = 0; kp < 4; ++kp) {
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4(st + k_off[nt][kp], b0, b1, b2, b3);
                    mma_bf16_16816(sc[nt], qa[2 * kp][0], qa[2 * kp][1], qa[2 * kp][2],
                                   qa[2 * kp][3], b0, b1);
                    mma_bf16_16816(sc[nt], qa[2 * kp + 1][0], qa[2 * kp + 1][1],
                                   qa[2 * kp + 1][2], qa[2 * kp + 1][3], b2, b3);
                }
            }

            // ---- online softmax (log2 domain), rows g and g+8 ----
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int tok = nt * 8 + 2 * t + j;
                    const bool ok = tok < fill;
                    sc[nt][j] = ok ? sc[nt][j] * p.scale_log2 : -INFINITY;
                    sc[nt][2 + j] = ok ? sc[nt][2 + j] * p.scale_log2 : -INFINITY;
                    mx0 = fmaxf(mx0, sc[nt][j]);
                    mx1 = fmaxf(mx1, sc[nt][2 + j]);
                }
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
            const float mn0 = fmaxf(m0, mx0);
            const float al0 = fast_exp2(m0 - mn0);
            m0 = mn0;
            float ps0 = 0.f;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    sc[nt][j] = fast_exp2(sc[nt][j] - mn0);
                    ps0 += sc[nt][j];
                }
            l0 = l0 * al0 + ps0;
            float al1 = 1.f;
            if constexpr (TWO_HALVES) {
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
                const float mn1 = fmaxf(m1, mx1);
                al1 = fast_exp2(m1 - mn1);
                m1 = mn1;
                float ps1 = 0.f;
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        sc[nt][2 + j] = fast_exp2(sc[nt][2 + j] - mn1);
                        ps1 += sc[nt][2 + j];
                    }
                l1 = l1 * al1 + ps1;
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                acc[i][0] *= al0;
                acc[i][1] *= al0;
                if constexpr (TWO_HALVES) {
                    acc[i][2] *= al1;
                    acc[i][3] *= al1;
                }
            }

            if constexpr (SPLIT) {  // K half consumed: hand it back before waiting for V
                __syncwarp();
                if (lane == 0) mbar_arrive(empty_bar + 8 * s);
                mbar_wait(full_bar + 8 * sv, phv);
            }

            // ---- O += P V ----
            const uint32_t pa0 = pack_bf16x2(sc[0][0], sc[0][1]);
            const uint32_t pa2 = pack_bf16x2(sc[1][0], sc[1][1]);
            const uint32_t pa1 = TWO_HALVES ? pack_bf16x2(sc[0][2], sc[0][3]) : 0u;
            const uint32_t pa3 = TWO_HALVES ? pack_bf16x2(sc[1][2], sc[1][3]) : 0u;
#pragma unroll
            for (int np = 0; np < 8; ++np) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(stv + v_off[np], b0, b1, b2, b3);
                mma_bf16_16816(acc[2 * np], pa0, pa1, pa2, pa3, b0, b1);
                mma_bf16_16816(acc[2 * np + 1], pa0, pa1, pa2, pa3, b2, b3);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty_bar + 8 * sv);
        }

        // ---- finalize the segment [seg_begin, seg_end) of shard r ----
        l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
        l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
        if constexpr (TWO_HALVES) {
            l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
            l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
        }
        if (p.trace && threadIdx.x == 0) p.trace[cta * 8 + 2] = k1_gtime();
        const bool complete = (seg_begin == r_first) && (seg_end == r_last);
        if (complete) {
            const float ln2 = 0.69314718055994530942f;
#pragma unroll
            for (int half = 0; half < (TWO_HALVES ? 2 : 1); ++half) {
                const bool real = half == 0 ? row0_real : row1_real;
                if (!real) continue;
                const int qh = h * G + g + 8 * half;
                const float l = half == 0 ? l0 : l1;
                const float m = half == 0 ? m0 : m1;
                const float inv = 1.f / l;
                float* o = row_out_c(p, r, rrt, C::HQ, C::D, ep) + qh * C::D + 2 * t;
#pragma unroll
                for (int nt = 0; nt < 16; ++nt)
                    *reinterpret_cast<float2*>(o + nt * 8) =
                        make_float2(acc[nt][2 * half] * inv, acc[nt][2 * half + 1] * inv);
                if (t == 0) row_lse_c(p, r, rrt, C::HQ, ep)[qh] = (m + __log2f(l)) * ln2;
            }
            if (p.xp) {
                named_bar_sync(1, NCT);
                if (threadIdx.x == 0) publish_row_c(p, rrt, ep);
            }
        } else {
            const int slot = 2 * cta + (seg_begin == p_begin ? 0 : 1);
#pragma unroll
            for (int half = 0; half < (TWO_HALVES ? 2 : 1); ++half) {
                const bool real = half == 0 ? row0_real : row1_real;
                if (!real) continue;
                const int qh = h * G + g + 8 * half;
                float* w = p.ws_acc + (static_cast<size_t>(slot) * C::HQ + qh) * C::D + 2 * t;
#pragma unroll
                for (int nt = 0; nt < 16; ++nt)
                    __stcg(reinterpret_cast<float2*>(w + nt * 8),
                           make_float2(acc[nt][2 * half], acc[nt][2 * half + 1]));
                if (t == 0)
                    __stcg(reinterpret_cast<float2*>(p.ws_ml) + (static_cast<size_t>(slot) * C::HQ + qh),
                           make_float2(half == 0 ? m0 : m1, half == 0 ? l0 : l1));
            }
            named_bar_sync(1, NCT);  // every warp's partial stores happen-before thread 0's release
            if (threadIdx.x == 0) {
                // P >= grid: every CTA of [a, b] holds pages of r; P < grid: every CTA holds at
                // most one page, so r has one part per page
                const int nparts = P < grid ? r_last - r_first
                                            : cta_of_page(r_last - 1, P, grid) - cta_of_page(r_first, P, grid) + 1;
                const int prev = atom_add_acq_rel_gpu(p.counters + r, 1);
                *last_flag = (prev == nparts - 1) ? 1 : 0;
            }
            named_bar_sync(1, NCT);
            if (p.trace && threadIdx.x == 0) p.trace[cta * 8 + 3] = k1_gtime();
            if (*last_flag) {
                // K9: merge the shard's partials in page order.  Part i is CTA a + i when
                // P >= grid (slot 2k, or 2k + 1 for CTA a when r starts inside its range), and the
                // CTA of page r_first + i when P < grid (one page per CTA, slot 2k).  Warp h owns
                // the G q-heads of kv-head h, lane j columns [4j, 4j+4).  Parts are taken 32 at a
                // time: each lane loads its part's (max, sum) of all G rows (kept in registers
                // when the shard has <= 32 parts), the live parts are a ballot, and the numerator
                // walks them U at a time with all U * G partial rows in flight.
                const bool sparse = P < grid;
                const int a = sparse ? 0 : cta_of_page(r_first, P, grid);
                const int nparts = sparse ? r_last - r_first : cta_of_page(r_last - 1, P, grid) - a + 1;
                const bool a_mid = !sparse && r_first != static_cast<int>(udiv64((int64_t)a * P, grid));
                const float ln2 = 0.69314718055994530942f;
                constexpr int U = G >= 16 ? 1 : (G >= 8 ? 2 : K9_U);
                auto slot_of_part = [&](int i) {
                    if (sparse) return 2 * cta_of_page(r_first + i, P, grid);
                    return 2 * (a + i) + ((i == 0 && a_mid) ? 1 : 0);
                };
                const float2* mlp = reinterpret_cast<const float2*>(p.ws_ml);
                float mmax[G];
                float2 ml0[G];  // this lane's part of the first 32
                const int sl0 = lane < nparts ? slot_of_part(lane) : 0;
#pragma unroll
                for (int row = 0; row < G; ++row) {
                    ml0[row] = lane < nparts ? __ldcg(mlp + (size_t)sl0 * C::HQ + h * G + row)
                                             : make_float2(-INFINITY, 0.f);
                    mmax[row] = ml0[row].x;
                }
                for (int base = 32; base < nparts; base += 32) {
                    if (base + lane < nparts) {
                        const size_t sl = slot_of_part(base + lane);
#pragma unroll
                        for (int row = 0; row < G; ++row)
                            mmax[row] = fmaxf(mmax[row], __ldcg(mlp + sl * C::HQ + h * G + row).x);
                    }
                }
#pragma unroll
                for (int row = 0; row < G; ++row)
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1)
                        mmax[row] = fmaxf(mmax[row], __shfl_xor_sync(0xffffffffu, mmax[row], o));
                float den[G];
                float4 num[G];
#pragma unroll
                for (int row = 0; row < G; ++row) {
                    den[row] = 0.f;
                    num[row] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
                for (int base = 0; base < nparts; base += 32) {
                    const bool live = base + lane < nparts;
                    const int sl = base == 0 ? sl0 : (live ? slot_of_part(base + lane) : 0);
                    float w[G];
#pragma unroll
                    for (int row = 0; row < G; ++row) {
                        w[row] = 0.f;
                        if (live) {
                            const float2 ml = base == 0 ? ml0[row] : __ldcg(mlp + (size_t)sl * C::HQ + h * G + row);
                            w[row] = fast_exp2(ml.x - mmax[row]);
                            den[row] += w[row] * ml.y;
                        }
                    }
                    unsigned mask = __ballot_sync(0xffffffffu, live);
                    while (mask) {
                        int src[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            src[u] = mask ? __ffs(mask) - 1 : -1;
                            mask &= mask - 1;
                        }
                        float4 v[U][G];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int su = __shfl_sync(0xffffffffu, sl, src[u] < 0 ? 0 : src[u]);
                            const float4* rowp =
                                reinterpret_cast<const float4*>(p.ws_acc + ((size_t)su * C::HQ + h * G) * C::D) + lane;
#pragma unroll
                            for (int row = 0; row < G; ++row)
                                v[u][row] = src[u] >= 0 ? __ldcg(rowp + row * (C::D / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int row = 0; row < G; ++row) {
                                const float wu = __shfl_sync(0xffffffffu, w[row], src[u] < 0 ? 0 : src[u]);
                                const float ww = src[u] >= 0 ? wu : 0.f;
                                num[row].x += ww * v[u][row].x;
                                num[row].y += ww * v[u][row].y;
                                num[row].z += ww * v[u][row].z;
                                num[row].w += ww * v[u][row].w;
                            }
                    }
                }
#pragma unroll
                for (int row = 0; row < G; ++row) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) den[row] += __shfl_xor_sync(0xffffffffu, den[row], o);
                    const int qh = h * G + row;
                    const float inv = 1.f / den[row];
                    float* o = row_out_c(p, r, rrt, C::HQ, C::D, ep) + qh * C::D;
                    reinterpret_cast<float4*>(o)[lane] =
                        make_float4(num[row].x * inv, num[row].y * inv, num[row].z * inv, num[row].w * inv);
                    if (lane == 0) row_lse_c(p, r, rrt, C::HQ, ep)[qh] = (mmax[row] + __log2f(den[row])) * ln2;
                }
                if (threadIdx.x == 0) p.counters[r] = 0;  // re-arm for the next launch / graph replay
                if (p.trace && threadIdx.x == 0) p.trace[cta * 8 + 4] = k1_gtime();
                if (p.xp) {
                    named_bar_sync(2, NCT);
                    if (threadIdx.x == 0) publish_row_c(p, rrt, ep);
                }
            }
        }
        ++r;
    }
    };  // attend
    if (p_begin < p_end) attend();

    if (p.fuse & FUSE_MERGE) {
        // K3: merge this CTA's M rows r = cta, cta + grid, ... once their |P_r| Res-route flags
        // carry epoch e; weights as lse_merge (attn_merge.hpp:86-100), zero-token shards
        // (LSE = -inf) weigh 0.  Every producer is co-resident (this kernel) or another GPU.
        const XchgPeers& x = *p.xp;
        __shared__ int32_t s_parts[PL_MAXK];
        const int M = x.W > 1 ? p.m_count[x.self] : 0;  // W = 1: every row was written final by K1
        for (int r = cta; r < M; r += gridDim.x) {
            const int k = p.m_k[r];
            if (k == 1 && p.m_kv[(size_t)r * PL_MAXK] == x.self) continue;  // written final by K1
            if (threadIdx.x < k) {
                const int s = p.m_kv[(size_t)r * PL_MAXK + threadIdx.x];
                s_parts[threadIdx.x] = s;
                wait_flag(xres_flag(x, x.self, ep) + (size_t)r * x.W + s, ep, x.wc,
                          (SITE_K3_RES << 24) | (s << 16) | (r & 0xffff));
            }
            named_bar_sync(1, NCT);
            const float* po = xres_o(x, x.self, ep) + (size_t)r * x.W * C::HQ * C::D;
            const float* pl = xres_lse(x, x.self, ep) + (size_t)r * x.W * C::HQ;
            // thread (head, 16-column quarter): C::HQ * 8 work items over NCT threads
            for (int wi = threadIdx.x; wi < C::HQ * (C::D / 16); wi += NCT) {
                const int qh = wi / (C::D / 16), c0 = (wi % (C::D / 16)) * 16;
                float mx = -INFINITY;
                for (int i = 0; i < k; ++i) mx = fmaxf(mx, __ldcg(pl + (size_t)s_parts[i] * C::HQ + qh));
                float4 acc[4] = {};
                float den = 0.f;
                for (int i = 0; i < k; ++i) {
                    const int s = s_parts[i];
                    const float l = __ldcg(pl + (size_t)s * C::HQ + qh);
                    const float wgt = l == -INFINITY ? 0.f : expf(l - mx);
                    den += wgt;
                    const float4* v = reinterpret_cast<const float4*>(po + ((size_t)s * C::HQ + qh) * C::D + c0);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float4 t4 = __ldcg(v + j);
                        acc[j].x += wgt * t4.x;
                        acc[j].y += wgt * t4.y;
                        acc[j].z += wgt * t4.z;
                        acc[j].w += wgt * t4.w;
                    }
                }
                const float inv = 1.f / den;
                float4* o = reinterpret_cast<float4*>(p.mout + ((size_t)r * C::HQ + qh) * C::D + c0);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    o[j] = make_float4(acc[j].x * inv, acc[j].y * inv, acc[j].z * inv, acc[j].w * inv);
                if (c0 == 0) p.mout_lse[(size_t)r * C::HQ + qh] = mx + logf(den);
            }
            named_bar_sync(1, NCT);  // s_parts is rewritten by the next row
        }
    }
    if (p.trace && threadIdx.x == 0) p.trace[cta * 8 + 5] = k1_gtime();
}

}  // namespace dcp
