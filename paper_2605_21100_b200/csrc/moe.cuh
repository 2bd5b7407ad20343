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
//   K4a moe_layout     one CTA: per destination rank a block-wide prefix over
//                      tokens gives each (token, rank) pair its slot in the
//                      peer's per-source region; counts are published first.
//   K4b moe_dispatch   one CTA per token: 16-byte stores of the hidden state
//                      into each destination's slot (+ expert ids / weights),
//                      then a per-slot arrival flag (st.release.sys = epoch).
//   K5a moe_receive    wait for counts and slots from every source, compact the
//                      received rows (source order, slot order) for the expert
//                      GEMMs.
//   K5b combine_put    each expert rank returns the gate-weighted sum over its
//                      local experts (bf16) to the token's home slot [t][rank].
//   K5c combine_reduce at home: sum the per-rank partials in ascending rank
//                      (= ascending expert) order into fp32.
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
    uint32_t* rx_flag[PL_MAXW];        // [W src][m_max]
    int32_t* rx_count[PL_MAXW];        // [W src]
    uint32_t* rx_count_flag[PL_MAXW];  // [W src]
    __nv_bfloat16* cb_y[PL_MAXW];      // [m_max][W dst][H]
    uint32_t* cb_flag[PL_MAXW];        // [m_max][W dst]
};

// K4a: slot of every (token, destination rank); counts published to peers.
static __global__ void __launch_bounds__(1024) moe_layout_kernel(const MoePeers* __restrict__ mp,
                                                                 const int32_t* __restrict__ topk_idx,
                                                                 const int32_t* __restrict__ m_count,
                                                                 int32_t* __restrict__ slot_tbl) {
    __shared__ int32_t wsum[32];
    __shared__ int32_t total[PL_MAXW];
    const MoePeers& p = *mp;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int M = *m_count;
    const int W = p.W;
    uint32_t mask = 0;
    if (t < M)
        for (int j = 0; j < p.topk; ++j) mask |= 1u << (topk_idx[t * p.topk + j] / p.e_per_rank);
    for (int d = 0; d < W; ++d) {
        const bool b = t < M && ((mask >> d) & 1u);
        const unsigned bal = __ballot_sync(0xffffffffu, b);
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        int base = 0;
        for (int w = 0; w < warp; ++w) base += wsum[w];
        if (t < M) slot_tbl[t * W + d] = b ? base + __popc(bal & ((1u << lane) - 1u)) : -1;
        if (t == 0) {
            int s = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += wsum[w];
            total[d] = s;
        }
        __syncthreads();
    }
    if (t < W) {
        const uint32_t ep = *p.epoch;
        p.rx_count[t][p.self] = total[t];
        st_release_sys(p.rx_count_flag[t] + p.self, ep);
    }
}

// K4b: one CTA per local token.
static __global__ void __launch_bounds__(128) moe_dispatch_kernel(const MoePeers* __restrict__ mp,
                                                                  const __nv_bfloat16* __restrict__ x,
                                                                  const int32_t* __restrict__ topk_idx,
                                                                  const float* __restrict__ topk_w,
                                                                  const int32_t* __restrict__ m_count,
                                                                  const int32_t* __restrict__ slot_tbl) {
    const MoePeers& p = *mp;
    const int t = blockIdx.x;
    if (t >= *m_count) return;
    const uint32_t ep = *p.epoch;
    const int W = p.W, H = p.H, vec = H / 8;
    const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)t * H);
    for (int d = 0; d < W; ++d) {
        const int slot = slot_tbl[t * W + d];
        if (slot < 0) continue;
        const size_t row = (size_t)p.self * p.m_max + slot;
        uint4* dst = reinterpret_cast<uint4*>(p.rx_x[d] + row * H);
        for (int i = threadIdx.x; i < vec; i += blockDim.x) dst[i] = __ldg(src + i);
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
        __syncthreads();
        if (threadIdx.x == 0) st_release_sys(p.rx_flag[d] + row, ep);
    }
}

// K5a: wait for every source, compact received rows in (source, slot) order.
static __global__ void __launch_bounds__(1024) moe_receive_kernel(const MoePeers* __restrict__ mp,
                                                                  __nv_bfloat16* __restrict__ x_rows,
                                                                  int32_t* __restrict__ meta_rows,
                                                                  int32_t* __restrict__ row_src,
                                                                  int32_t* __restrict__ counts) {
    __shared__ int32_t cnt[PL_MAXW], off[PL_MAXW + 1];
    const MoePeers& p = *mp;
    const uint32_t ep = *p.epoch;
    const int W = p.W, H = p.H;
    if (threadIdx.x < W) {
        wait_flag(p.rx_count_flag[p.self] + threadIdx.x, ep);
        cnt[threadIdx.x] = *((volatile int32_t*)p.rx_count[p.self] + threadIdx.x);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        off[0] = 0;
        for (int s = 0; s < W; ++s) off[s + 1] = off[s] + cnt[s];
        for (int s = 0; s < W; ++s) counts[s] = cnt[s];
    }
    __syncthreads();
    const int R = off[W];
    // one warp per received row
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int r = warp; r < R; r += nw) {
        int s = 0;
        while (off[s + 1] <= r) ++s;
        const int slot = r - off[s];
        const size_t row = (size_t)s * p.m_max + slot;
        if (lane == 0) wait_flag(p.rx_flag[p.self] + row, ep);
        __syncwarp();
        const uint4* src = reinterpret_cast<const uint4*>(p.rx_x[p.self] + row * H);
        uint4* dst = reinterpret_cast<uint4*>(x_rows + (size_t)r * H);
        for (int i = lane; i < H / 8; i += 32) dst[i] = __ldcg(src + i);
        for (int i = lane; i < p.meta; i += 32) meta_rows[(size_t)r * p.meta + i] = __ldcg(p.rx_meta[p.self] + row * p.meta + i);
        if (lane == 0) row_src[r] = s;
    }
}

// K5b: return each received row's partial sum to the token's home.
static __global__ void __launch_bounds__(128) moe_combine_put_kernel(const MoePeers* __restrict__ mp,
                                                                     const __nv_bfloat16* __restrict__ y_rows,
                                                                     const int32_t* __restrict__ meta_rows,
                                                                     const int32_t* __restrict__ row_src,
                                                                     const int32_t* __restrict__ counts) {
    const MoePeers& p = *mp;
    int R = 0;
    for (int s = 0; s < p.W; ++s) R += counts[s];
    const int r = blockIdx.x;
    if (r >= R) return;
    const uint32_t ep = *p.epoch;
    const int s = row_src[r];
    const int t = meta_rows[(size_t)r * p.meta];
    const int H = p.H;
    const uint4* src = reinterpret_cast<const uint4*>(y_rows + (size_t)r * H);
    uint4* dst = reinterpret_cast<uint4*>(p.cb_y[s] + ((size_t)t * p.W + p.self) * H);
    for (int i = threadIdx.x; i < H / 8; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
    if (threadIdx.x == 0) st_release_sys(p.cb_flag[s] + (size_t)t * p.W + p.self, ep);
}

// K5c: at home, sum the partials of every destination rank in ascending order.
static __global__ void __launch_bounds__(256) moe_combine_reduce_kernel(const MoePeers* __restrict__ mp,
                                                                        const int32_t* __restrict__ m_count,
                                                                        const int32_t* __restrict__ slot_tbl,
                                                                        float* __restrict__ out) {
    const MoePeers& p = *mp;
    const int t = blockIdx.x;
    if (t >= *m_count) return;
    const uint32_t ep = *p.epoch;
    const int W = p.W, H = p.H;
    if (threadIdx.x < W && slot_tbl[t * W + threadIdx.x] >= 0)
        wait_flag(p.cb_flag[p.self] + (size_t)t * W + threadIdx.x, ep);
    __syncthreads();
    for (int h2 = threadIdx.x; h2 < H / 2; h2 += blockDim.x) {
        float a = 0.f, b = 0.f;
        for (int d = 0; d < W; ++d) {
            if (slot_tbl[t * W + d] < 0) continue;
            const __nv_bfloat162 v =
                __ldcg(reinterpret_cast<const __nv_bfloat162*>(p.cb_y[p.self] + ((size_t)t * W + d) * H) + h2);
            const float2 f = __bfloat1622float2(v);
            a += f.x;
            b += f.y;
        }
        reinterpret_cast<float2*>(out + (size_t)t * H)[h2] = make_float2(a, b);
    }
}

}  // namespace dcp

namespace dcp {
static __global__ void epoch_bump_kernel_moe(uint32_t* epoch) { *epoch += 1; }
}  // namespace dcp
