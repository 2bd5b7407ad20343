// SPDX-License-Identifier: Apache-2.0
//
// K4 / K5: MoE token dispatch / combine over NVLink peer pools (north_star
// subsystem 3).  The reference has no MoE code: its only MoE surface is the
// per-instance list of MoE-bound requests (BindingConfig::moe_bound,
// routing.hpp:18-19; B_s, scheduler.cpp:288).  Here that list is the token
// order of each instance: token t of instance m is the t-th request of m's
// M list, and the tokens' top-k experts decide where they go.  Counts are
// known a priori from the gating, so there is no runtime handshake
// (PAPER.md:869).
//
//   K4  moe_dispatch   CTAs (chunk, destination rank): a block-wide ballot prefix
//                      over the tokens gives each (token, rank) its slot in the
//                      peer's per-source region; 16-byte stores of the hidden
//                      states routed to that rank (+ expert ids / weights); the
//                      last chunk CTA of a destination publishes the count and one
//                      (source -> destination) flag (st.release.sys = epoch) after
//                      every chunk's system fence: W flags per instance and step.
//   K5a moe_receive    wait for counts and slots from every source, compact the
//                      received rows (source order, slot order) for the expert
//                      GEMMs.
//   K5b combine_put    CTAs (chunk, home rank): each expert rank returns the
//                      gate-weighted sum over its local experts (bf16) to the
//                      token's home slot [t][rank]; one (rank -> home) flag per
//                      home, published like K4b's.
//   K5c combine_reduce at home: wait for every rank's flag, sum the per-rank
//                      partials in ascending rank (= ascending expert) order into fp32.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>

#include "exchange.cuh"
#include "limits.cuh"

namespace dcp {

constexpr int MOE_MAXK = 16;

struct MoePeers {
    int32_t W, self, H, topk, e_per_rank, m_max, meta;  // meta = 2 + 2*topk int32 per row
    uint32_t* epoch;
    __nv_bfloat16* rx_x[PL_MAXW];      // [W src][m_max][H]
    int32_t* rx_meta[PL_MAXW];         // [W src][m_max][meta]: src token, n_local, (expert, weight bits)*
    uint32_t* rx_flag[PL_MAXW];        // [W src]: all of src's rows for this rank have landed
    int32_t* rx_count[PL_MAXW];        // [W src]
    __nv_bfloat16* cb_y[PL_MAXW];      // [m_max][W dst][H]
    uint32_t* cb_flag[PL_MAXW];        // [W dst]: all of dst's partials for this home have landed
    int32_t* disp_done;                // [W dst] local: dispatch chunk CTAs finished (self-resetting)
    int32_t* cb_done;                  // [W home] local: combine chunk CTAs finished (self-resetting)
    int32_t chunks;                    // CTAs per destination / home rank
};

// Copy one row of `nvec` 16-byte vectors with the block, UNROLL loads in flight per thread
// before their stores (a row copy is latency-bound otherwise).
template <int UNROLL = 4, bool CG = false>
__device__ __forceinline__ void copy_row(uint4* __restrict__ dst, const uint4* __restrict__ src, int nvec) {
    for (int base = threadIdx.x; base < nvec; base += UNROLL * blockDim.x) {
        uint4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const int i = base + u * blockDim.x;
            if (i < nvec) v[u] = CG ? __ldcg(src + i) : __ldg(src + i);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const int i = base + u * blockDim.x;
            if (i < nvec) dst[i] = v[u];
        }
    }
}

// Chunk CTA epilogue: after this CTA's stores, the last of `chunks` CTAs publishes `flag`.
// Every CTA fences system-wide before its ticket, so the last one's release covers all.
__device__ __forceinline__ void moe_chunk_done(int32_t* done, int chunks, uint32_t* flag, uint32_t ep) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(done, 1) == chunks - 1) {
            atomicExch(done, 0);
            st_release_sys(flag, ep);
        }
    }
}

// K4: CTA (chunk c, destination d).  Every CTA of destination d scans the tokens (block-wide
// ballot prefix) for their slots in d's region; chunk c sends tokens t = c, c + chunks, ...
// routed to d; the last chunk CTA publishes the count and one (source -> d) flag.  Chunk 0
// also records the slot table for the combine.
static __global__ void __launch_bounds__(128) moe_dispatch_kernel(const MoePeers* __restrict__ mp,
                                                                  const __nv_bfloat16* __restrict__ x,
                                                                  const int32_t* __restrict__ topk_idx,
                                                                  const float* __restrict__ topk_w,
                                                                  const int32_t* __restrict__ m_count,
                                                                  int32_t* __restrict__ slot_tbl) {
    __shared__ int32_t wsum[4];
    __shared__ int16_t mine_t[1024], mine_s[1024];
    __shared__ int32_t n_mine;
    const MoePeers& p = *mp;
    const int d = blockIdx.y, c = blockIdx.x, M = *m_count;
    const uint32_t ep = *p.epoch;
    const int W = p.W, H = p.H, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) n_mine = 0;
    __syncthreads();  // the scan loop below holds the other barriers, and it is empty when M == 0
    int carry = 0;
    for (int t0 = 0; t0 < M; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        bool routed = false;
        if (t < M)
            for (int j = 0; j < p.topk; ++j) routed |= topk_idx[t * p.topk + j] / p.e_per_rank == d;
        const unsigned bal = __ballot_sync(0xffffffffu, routed);
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        int base = carry;
        for (int w = 0; w < warp; ++w) base += wsum[w];
        const int slot = base + __popc(bal & ((1u << lane) - 1u));
        if (t < M && c == 0) slot_tbl[t * W + d] = routed ? slot : -1;
        if (routed && t % p.chunks == c) {
            const int k = atomicAdd(&n_mine, 1);
            mine_t[k] = static_cast<int16_t>(t);
            mine_s[k] = static_cast<int16_t>(slot);
        }
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) carry += wsum[w];
        __syncthreads();
    }
    for (int k = 0; k < n_mine; ++k) {
        const int t = mine_t[k], slot = mine_s[k];
        const size_t row = (size_t)p.self * p.m_max + slot;
        copy_row(reinterpret_cast<uint4*>(p.rx_x[d] + row * H), reinterpret_cast<const uint4*>(x + (size_t)t * H), H / 8);
        if (threadIdx.x == 0) {
            int32_t* meta = p.rx_meta[d] + row * p.meta;
            int n = 0;
            for (int j = 0; j < p.topk; ++j) {
                const int e = topk_idx[t * p.topk + j];
                if (e / p.e_per_rank != d) continue;
                meta[2 + 2 * n] = e;
                meta[3 + 2 * n] = __float_as_int(topk_w[t * p.topk + j]);
                ++n;
            }
            meta[0] = t;
            meta[1] = n;
        }
    }
    // last chunk: count, then the flag (covers every chunk's rows, see moe_chunk_done)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(p.disp_done + d, 1) == p.chunks - 1) {
            atomicExch(p.disp_done + d, 0);
            p.rx_count[d][p.self] = carry;
            st_release_sys(p.rx_flag[d] + p.self, ep);
        }
    }
}

// K5a: wait for every source, compact received rows in (source, slot) order.  Grid-wide:
// every CTA derives the per-source offsets from the published counts, then its warp groups
// copy rows r = group_global, + total_groups, ...
static __global__ void __launch_bounds__(256) moe_receive_kernel(const MoePeers* __restrict__ mp,
                                                                 __nv_bfloat16* __restrict__ x_rows,
                                                                 int32_t* __restrict__ meta_rows,
                                                                 int32_t* __restrict__ row_src,
                                                                 int32_t* __restrict__ counts) {
    __shared__ int32_t cnt[PL_MAXW], off[PL_MAXW + 1];
    const MoePeers& p = *mp;
    const uint32_t ep = *p.epoch;
    const int W = p.W, H = p.H;
    if (threadIdx.x < W) {
        wait_flag(p.rx_flag[p.self] + threadIdx.x, ep);
        cnt[threadIdx.x] = *((volatile int32_t*)p.rx_count[p.self] + threadIdx.x);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        off[0] = 0;
        for (int s = 0; s < W; ++s) off[s + 1] = off[s] + cnt[s];
        if (blockIdx.x == 0)
            for (int s = 0; s < W; ++s) counts[s] = cnt[s];
    }
    __syncthreads();
    const int R = off[W];
    // a group of wpr warps per row, wpr ~ vectors / 128 (capped at the CTA's 8 warps): a
    // 7,168-wide row (896 vectors) takes the whole CTA and is in flight at once, a 2,048-wide
    // row two warps (one warp per row took H / 1,024 dependent load rounds)
    const int nvec = H / 8;
    const int wpr = nvec > 512 ? 8 : nvec > 256 ? 4 : nvec > 128 ? 2 : 1;
    const int gsz = 32 * wpr, groups = (blockDim.x >> 5) / wpr;
    const int grp = (threadIdx.x >> 5) / wpr, gt = threadIdx.x % gsz;
    for (int r = blockIdx.x * groups + grp; r < R; r += gridDim.x * groups) {
        int s = 0;
        while (off[s + 1] <= r) ++s;
        const int slot = r - off[s];
        const size_t row = (size_t)s * p.m_max + slot;
        const uint4* src = reinterpret_cast<const uint4*>(p.rx_x[p.self] + row * H);
        uint4* dst = reinterpret_cast<uint4*>(x_rows + (size_t)r * H);
        for (int base = gt; base < nvec; base += 4 * gsz) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (base + gsz * u < nvec) v[u] = __ldcg(src + base + gsz * u);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (base + gsz * u < nvec) dst[base + gsz * u] = v[u];
        }
        for (int i = gt; i < p.meta; i += gsz)
            meta_rows[(size_t)r * p.meta + i] = __ldcg(p.rx_meta[p.self] + row * p.meta + i);
        if (gt == 0) row_src[r] = s;
    }
}

// K5b: CTA (chunk c, home s) returns received rows r = off[s] + c, + chunks, ... (the rows that
// came from s, compacted contiguously by K5a) to their tokens' home slots.
static __global__ void __launch_bounds__(128) moe_combine_put_kernel(const MoePeers* __restrict__ mp,
                                                                     const __nv_bfloat16* __restrict__ y_rows,
                                                                     const int32_t* __restrict__ meta_rows,
                                                                     const int32_t* __restrict__ counts) {
    const MoePeers& p = *mp;
    const int s = blockIdx.y;
    int off = 0;
    for (int k = 0; k < s; ++k) off += counts[k];
    const int n = counts[s];
    const uint32_t ep = *p.epoch;
    const int H = p.H;
    for (int i = blockIdx.x; i < n; i += p.chunks) {
        const int r = off + i;
        const int t = meta_rows[(size_t)r * p.meta];
        copy_row(reinterpret_cast<uint4*>(p.cb_y[s] + ((size_t)t * p.W + p.self) * H),
                 reinterpret_cast<const uint4*>(y_rows + (size_t)r * H), H / 8);
    }
    moe_chunk_done(p.cb_done + s, p.chunks, p.cb_flag[s] + p.self, ep);
}

// K5c: at home, sum the partials of every destination rank in ascending order.  CTA (token t,
// hidden chunk); each thread owns 4 consecutive columns and loads all ranks' partials before
// adding them (the W loads are in flight together).
static __global__ void __launch_bounds__(256) moe_combine_reduce_kernel(const MoePeers* __restrict__ mp,
                                                                        const int32_t* __restrict__ m_count,
                                                                        const int32_t* __restrict__ slot_tbl,
                                                                        float* __restrict__ out) {
    const MoePeers& p = *mp;
    const int t = blockIdx.x;
    if (t >= *m_count) return;
    const uint32_t ep = *p.epoch;
    const int W = p.W, H = p.H;
    if (threadIdx.x < W) wait_flag(p.cb_flag[p.self] + threadIdx.x, ep);
    __syncthreads();
    const int q = blockIdx.y * blockDim.x + threadIdx.x;  // 4-column group
    if (4 * q >= H) return;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    uint2 v[PL_MAXW];
#pragma unroll 8
    for (int d = 0; d < W; ++d)
        if (slot_tbl[t * W + d] >= 0)
            v[d] = __ldcg(reinterpret_cast<const uint2*>(p.cb_y[p.self] + ((size_t)t * W + d) * H) + q);
#pragma unroll 8
    for (int d = 0; d < W; ++d) {
        if (slot_tbl[t * W + d] < 0) continue;
        const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v[d].x));
        const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v[d].y));
        a0 += lo.x;
        a1 += lo.y;
        a2 += hi.x;
        a3 += hi.y;
    }
    reinterpret_cast<float4*>(out + (size_t)t * H)[q] = make_float4(a0, a1, a2, a3);
}

}  // namespace dcp

namespace dcp {
static __global__ void epoch_bump_kernel_moe(uint32_t* epoch) { *epoch += 1; }
}  // namespace dcp
