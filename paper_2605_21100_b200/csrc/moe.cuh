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
//   K4  moe_dispatch   every CTA derives the layout (each token's destination
//                      ranks, its slot in each destination's per-source region)
//                      from the gating in shared memory; CTA c then sends tokens
//                      c, c + C, ...: the hidden state is loaded ONCE into
//                      registers and stored to every destination rank it is
//                      routed to (16-byte vectors, remote NVLink stores on a
//                      multi-GPU node).  Completion (MOE_SINGLE_RELEASE, the
//                      default): the CTAs meet on a gpu-scope ticket; the last
//                      one issues one system fence and adds each destination's
//                      row count to its arrival counter (relaxed system-scope
//                      reds); CTA 0 publishes the count record {epoch, count}
//                      and the cumulative row target.  No per-row flag.
//   K5a moe_receive    wait, per source, for the count record and for the
//                      arrival counter to reach its target; the rows stay in
//                      the pool's per-source regions [W][m_max][H] (the expert
//                      stage reads them there), or are compacted (legacy
//                      dcp_moe_receive).
//   K5b combine_put    one warp per received row returns its y row (gate-weighted
//                      sum over this rank's experts) to the token's home slot
//                      [t][rank]; arrival counted like K4.
//   fused forms        (one instance per process / GPU) K4 + K5a and K5b + K5c in
//                      one launch each: dcp_moe_step_dispatch_recv,
//                      dcp_moe_combine_fused.
//   K5c combine_reduce at home: wait for every rank's counter to reach the rows it
//                      owes (known from the home's own gating), sum the per-rank
//                      partials in ascending rank (= ascending expert) order, fp32.
//
// Counters are cumulative per (parity, source) and never reset: a waiter compares
// against a cumulative target in serial-number order, so any number of CTAs can
// wait on them.  Buffers are double-buffered by the step epoch's parity and the
// step fence of exchange.cuh keeps every instance within one step of its peers.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>

#include "exchange.cuh"
#include "limits.cuh"
#include "ptx.cuh"

namespace dcp {

constexpr int MOE_MAXK = 16;
#ifndef MOE_K5B_WARP
#define MOE_K5B_WARP 1  // K5b: one warp per row (1) or one CTA per row (0)
#endif
#ifndef MOE_K4_FENCE_FIRST
#define MOE_K4_FENCE_FIRST 1  // K4: warp 0 runs the step fence while warps 1.. build the token masks (1)
#endif
#ifndef MOE_K4_PRELOAD
#define MOE_K4_PRELOAD 1  // K4: load the CTA's first token row before the layout / fence
#endif
#ifndef MOE_SINGLE_RELEASE
#define MOE_SINGLE_RELEASE 1  // K4 / K5b: CTAs meet on a gpu-scope ticket; the last one issues ONE system fence
#endif                        // and the per-destination row counts (instead of a red.release.sys per CTA)
constexpr int MOE_THREADS = 256;

struct MoePeers {
    int32_t W, self, H, topk, e_per_rank, m_max, meta;  // meta = 2 + 2*topk int32 per row
    uint32_t* epoch;
    WaitCtl wc;
    char* base[PL_MAXW];
    // pool layout, per parity p (at off_* + p * sz_*):
    //   rx_x     [W src][m_max][H] bf16
    //   rx_meta  [W src][m_max][meta] int32: src token, n_local, (expert, weight bits) * n_local
    //   rx_cnt   [W src][2] u64: {epoch << 32 | count}, cumulative row target
    //   rx_arr   [W src] u32 cumulative rows landed
    //   cb_y     [m_max][W rank][H] bf16
    //   cb_arr   [W rank] u32 cumulative rows landed
    //   done     u32 (step fence)
    uint64_t off_rx_x, off_rx_meta, off_rx_cnt, off_rx_arr, off_cb_y, off_cb_arr, off_done;
    uint64_t sz_rx_x, sz_rx_meta, sz_rx_cnt, sz_rx_arr, sz_cb_y, sz_cb_arr;
    // local
    int32_t* slot_tbl;     // [m_max][W] home: token t's slot at rank d, -1 = not routed there
    uint32_t* cum_sent;    // [2][W] rows sent to each destination, per parity (cumulative)
    uint32_t* cb_target;   // [2][W] rows each rank owes this home, per parity (cumulative)
    int32_t* counts;       // [W] rows received from each source this step
    int32_t* offs;         // [W + 1] exclusive prefix of counts
    int32_t chunks;        // CTAs of K4 / K5b
    int32_t* exit_ticket;  // K4 with the step fence folded in: grid exit counter
};

template <class T>
__device__ __forceinline__ T* mp_at(const MoePeers& p, int s, uint64_t off, uint64_t sz, uint32_t ep) {
    return reinterpret_cast<T*>(p.base[s] + off + (ep & 1) * sz);
}
__device__ __forceinline__ __nv_bfloat16* rx_x(const MoePeers& p, int s, uint32_t ep) {
    return mp_at<__nv_bfloat16>(p, s, p.off_rx_x, p.sz_rx_x, ep);
}
__device__ __forceinline__ int32_t* rx_meta(const MoePeers& p, int s, uint32_t ep) {
    return mp_at<int32_t>(p, s, p.off_rx_meta, p.sz_rx_meta, ep);
}
__device__ __forceinline__ unsigned long long* rx_cnt(const MoePeers& p, int s, uint32_t ep) {
    return mp_at<unsigned long long>(p, s, p.off_rx_cnt, p.sz_rx_cnt, ep);
}
__device__ __forceinline__ uint32_t* rx_arr(const MoePeers& p, int s, uint32_t ep) {
    return mp_at<uint32_t>(p, s, p.off_rx_arr, p.sz_rx_arr, ep);
}
__device__ __forceinline__ __nv_bfloat16* cb_y(const MoePeers& p, int s, uint32_t ep) {
    return mp_at<__nv_bfloat16>(p, s, p.off_cb_y, p.sz_cb_y, ep);
}
__device__ __forceinline__ uint32_t* cb_arr(const MoePeers& p, int s, uint32_t ep) {
    return mp_at<uint32_t>(p, s, p.off_cb_arr, p.sz_cb_arr, ep);
}
__device__ __forceinline__ uint32_t* moe_done(const MoePeers& p, int s) {
    return reinterpret_cast<uint32_t*>(p.base[s] + p.off_done);
}

__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Wait for source s's count record of epoch ep and for all of its rows; returns the count.
// The record {epoch << 32 | count, cumulative row target} (one 16-byte acquire load) and the
// cumulative arrival counter are polled in the same round: when the record carries ep and the
// counter has reached its target, every row is visible (the counter's releases cover them).
// One L2 round trip when the rows are already there, instead of three dependent ones.
__device__ __forceinline__ int moe_wait_source(const MoePeers& p, int s, uint32_t ep) {
    const unsigned long long* rec = rx_cnt(p, p.self, ep) + 2 * s;
    const uint32_t* arr = rx_arr(p, p.self, ep) + s;
    const uint32_t where = (SITE_MOE_RX << 24) | (s << 16);
    unsigned long long a = 0, tgt = 0;
    wait_until(
        [&](uint32_t& seen) {
            uint32_t c;
            asm volatile("ld.acquire.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(tgt) : "l"(rec) : "memory");
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(c) : "l"(arr) : "memory");
            seen = static_cast<uint32_t>(a >> 32);
            if (seen != ep) return false;
            seen = c;
            return static_cast<int32_t>(c - static_cast<uint32_t>(tgt)) >= 0;
        },
        ep, p.wc, where);
    return static_cast<int>(a & 0xffffffffu);
}

static __global__ void __launch_bounds__(32) moe_begin_step_kernel(const __grid_constant__ MoePeers p) {
    pdl_trigger();  // MoE launches are PDL-chained (capi_moe.cu)
    pdl_wait();
    step_fence(p.epoch, [&](int s) { return moe_done(p, s); }, p.W, p.self, p.wc);
}

// K5a body (one warp): lane s waits for source s's count record and rows of epoch ep, then the
// per-source counts and their exclusive prefix go to the device (graph-capturable, no host copy).
__device__ __forceinline__ void receive_counts_warp(const MoePeers& p, uint32_t ep) {
    const int lane = threadIdx.x & 31;
    int c = 0;
    if (lane < p.W) c = moe_wait_source(p, lane, ep);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane < p.W) {
        p.counts[lane] = c;
        p.offs[lane + 1] = incl;
    }
    if (lane == 0) p.offs[0] = 0;
}

// K4.  grid = chunks, block = MOE_THREADS; dynamic smem = m_max * (W + 1) * 4 bytes.
// with_fence: this launch is also the step's begin_step (the step fence of exchange.cuh before
// the first peer store; epoch e = *epoch + 1, advanced by the last CTA out), one launch per step.
static __global__ void __launch_bounds__(MOE_THREADS) moe_dispatch_kernel(const __grid_constant__ MoePeers p,
                                                                          const __nv_bfloat16* __restrict__ x,
                                                                          const int32_t* __restrict__ topk_idx,
                                                                          const float* __restrict__ topk_w,
                                                                          const int32_t* __restrict__ m_count,
                                                                          int with_fence, int with_recv) {
    pdl_trigger();  // MoE launches are PDL-chained (capi_moe.cu)
    pdl_wait();
    extern __shared__ int32_t sm[];
    const int W = p.W, H = p.H, K = p.topk, M = *m_count;
    int32_t* s_mask = sm;               // [M] destination-rank bitmask of each token
    int32_t* s_slot = sm + p.m_max;     // [M][W] slot at each destination (-1 = not routed)
    __shared__ int32_t s_count[PL_MAXW], s_sent[PL_MAXW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t ep = *p.epoch + (with_fence ? 1u : 0u);
    constexpr int NW = MOE_THREADS / 32;
    constexpr int VPT = 4;  // 16-byte vectors in registers per thread per pass (4 x 256 x 16 B = 16 KB)
    const int nvec = H / 8;
    uint4 v[VPT];
#if MOE_K4_PRELOAD
    if (static_cast<int>(blockIdx.x) < M) {
        const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)blockIdx.x * H);
#pragma unroll
        for (int u = 0; u < VPT; ++u)
            if (u * MOE_THREADS + tid < nvec) v[u] = __ldg(src + u * MOE_THREADS + tid);
    }
#endif
#if MOE_K4_FENCE_FIRST
    if (with_fence && warp == 0) {
        if (blockIdx.x == 0 && lane == 0) st_relaxed_sys(moe_done(p, p.self), ep - 1);
        for (int s = lane; s < W; s += 32)
            if (s != p.self) wait_flag(moe_done(p, s), ep - 2, p.wc, (SITE_FENCE << 24) | (s << 16), true);
    }
    for (int t = tid - 32; t < M; t += MOE_THREADS - 32) {
        if (t < 0) break;
#else
    for (int t = tid; t < M; t += MOE_THREADS) {
#endif
        uint32_t m = 0;
        for (int j = 0; j < K; ++j) m |= 1u << (__ldg(topk_idx + t * K + j) / p.e_per_rank);
        s_mask[t] = static_cast<int32_t>(m);
    }
    if (tid < PL_MAXW) s_sent[tid] = 0;
    __syncthreads();
    // slots: warp d scans the tokens for destination d (ballot prefix, ascending token order)
    for (int d = warp; d < W; d += NW) {
        int carry = 0;
        for (int t0 = 0; t0 < M; t0 += 32) {
            const int t = t0 + lane;
            const bool r = t < M && ((s_mask[t] >> d) & 1);
            const unsigned b = __ballot_sync(0xffffffffu, r);
            if (t < M) s_slot[t * W + d] = r ? carry + __popc(b & ((1u << lane) - 1u)) : -1;
            carry += __popc(b);
        }
        if (lane == 0) s_count[d] = carry;
    }
    if (!MOE_K4_FENCE_FIRST && with_fence && warp == 0) {
        if (blockIdx.x == 0 && lane == 0) st_relaxed_sys(moe_done(p, p.self), ep - 1);
        for (int s = lane; s < W; s += 32)
            if (s != p.self) wait_flag(moe_done(p, s), ep - 2, p.wc, (SITE_FENCE << 24) | (s << 16), true);
    }
    __syncthreads();
    if (blockIdx.x == 0) {
        for (int i = tid; i < M * W; i += MOE_THREADS) p.slot_tbl[i] = s_slot[i];
        if (tid < W) {
            const int d = tid, c = s_count[d];
            // the home expects c combine rows back from rank d (K5c); rank d gets c rows from us
            p.cb_target[(ep & 1) * W + d] += c;
            const uint32_t cum = (p.cum_sent[(ep & 1) * W + d] += c);
            unsigned long long* rec = rx_cnt(p, d, ep) + 2 * p.self;
            __stcg(rec + 1, static_cast<unsigned long long>(cum));
            st_release_sys_u64(rec, (static_cast<unsigned long long>(ep) << 32) | static_cast<uint32_t>(c));
        }
    }
    // rows: CTA c sends tokens c, c + C, ...; each token's hidden state is read once and
    // stored to all of its destination ranks.
    for (int t = blockIdx.x; t < M; t += gridDim.x) {
        const uint32_t mask = static_cast<uint32_t>(s_mask[t]);
        const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)t * H);
        for (int v0 = 0; v0 < nvec; v0 += VPT * MOE_THREADS) {
            if (!MOE_K4_PRELOAD || t != static_cast<int>(blockIdx.x) || v0 != 0) {
#pragma unroll
                for (int u = 0; u < VPT; ++u) {
                    const int i = v0 + u * MOE_THREADS + tid;
                    if (i < nvec) v[u] = __ldg(src + i);
                }
            }
            for (uint32_t mm = mask; mm; mm &= mm - 1) {
                const int d = __ffs(mm) - 1;
                const size_t row = (size_t)p.self * p.m_max + s_slot[t * W + d];
                uint4* dst = reinterpret_cast<uint4*>(rx_x(p, d, ep) + row * H);
#pragma unroll
                for (int u = 0; u < VPT; ++u) {
                    const int i = v0 + u * MOE_THREADS + tid;
                    if (i < nvec) dst[i] = v[u];
                }
            }
        }
        // meta rows: lane d of warp 0 writes destination d's
        if (tid < W && ((mask >> tid) & 1)) {
            const int d = tid;
            int32_t* meta = rx_meta(p, d, ep) + ((size_t)p.self * p.m_max + s_slot[t * W + d]) * p.meta;
            int n = 0;
            for (int j = 0; j < K; ++j) {
                const int e = __ldg(topk_idx + t * K + j);
                if (e / p.e_per_rank != d) continue;
                meta[2 + 2 * n] = e;
                meta[3 + 2 * n] = __float_as_int(__ldg(topk_w + t * K + j));
                ++n;
            }
            meta[0] = t;
            meta[1] = n;
            ++s_sent[d];
        }
    }
    __syncthreads();
#if MOE_SINGLE_RELEASE
    // The CTAs meet on a gpu-scope acq_rel ticket; the last one has acquired every CTA's row stores
    // and publishes them with one system fence (release cumulativity) and relaxed count adds.
    __shared__ int32_t s_last;
    if (tid == 0) {
        int old;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(p.exit_ticket) : "memory");
        s_last = old == static_cast<int>(gridDim.x) - 1;
        if (s_last) {
            *p.exit_ticket = 0;
            asm volatile("fence.acq_rel.sys;" ::: "memory");
            for (int d = 0; d < W; ++d)
                if (s_count[d]) asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(rx_arr(p, d, ep) + p.self),
                                             "r"(s_count[d]) : "memory");
            if (with_fence) *p.epoch = ep;
        }
    }
    if (with_recv) {
        // fused K5a (one instance per process / GPU only): the last CTA's warp 0 waits for every
        // source's rows of this epoch and writes the counts the expert stage reads
        __syncthreads();
        if (s_last && warp == 0) receive_counts_warp(p, ep);
    }
    return;
#endif
    // one release per (CTA, destination) covers every row this CTA stored there
    if (tid < W && s_sent[tid]) red_release_sys_add(rx_arr(p, tid, ep) + p.self, s_sent[tid]);
    if (with_fence && tid == 0) {
        int old;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(p.exit_ticket) : "memory");
        if (old == static_cast<int>(gridDim.x) - 1) {
            *p.exit_ticket = 0;
            *p.epoch = ep;
        }
    }
}

// K5a (region mode): one warp; lane s waits for source s, then counts and offsets.
static __global__ void __launch_bounds__(32) moe_receive_counts_kernel(const __grid_constant__ MoePeers p) {
    pdl_trigger();  // MoE launches are PDL-chained (capi_moe.cu)
    pdl_wait();
    receive_counts_warp(p, *p.epoch);
}

// K5a (compact mode, legacy dcp_moe_receive): every CTA waits for every source, then warp
// groups copy rows r = group_global, + total_groups, ... in (source, slot) order.
static __global__ void __launch_bounds__(256) moe_receive_compact_kernel(const __grid_constant__ MoePeers p,
                                                                         __nv_bfloat16* __restrict__ x_rows,
                                                                         int32_t* __restrict__ meta_rows) {
    pdl_trigger();  // MoE launches are PDL-chained (capi_moe.cu)
    pdl_wait();
    __shared__ int32_t cnt[PL_MAXW], off[PL_MAXW + 1];
    const uint32_t ep = *p.epoch;
    const int W = p.W, H = p.H;
    if (threadIdx.x < W) cnt[threadIdx.x] = moe_wait_source(p, threadIdx.x, ep);
    __syncthreads();
    if (threadIdx.x == 0) {
        off[0] = 0;
        for (int s = 0; s < W; ++s) off[s + 1] = off[s] + cnt[s];
        if (blockIdx.x == 0) {
            for (int s = 0; s < W; ++s) p.counts[s] = cnt[s];
            for (int s = 0; s <= W; ++s) p.offs[s] = off[s];
        }
    }
    __syncthreads();
    const int R = off[W];
    const int nvec = H / 8;
    const int wpr = nvec > 512 ? 8 : nvec > 256 ? 4 : nvec > 128 ? 2 : 1;
    const int gsz = 32 * wpr, groups = (blockDim.x >> 5) / wpr;
    const int grp = (threadIdx.x >> 5) / wpr, gt = threadIdx.x % gsz;
    const __nv_bfloat16* rx = rx_x(p, p.self, ep);
    const int32_t* rm = rx_meta(p, p.self, ep);
    for (int r = blockIdx.x * groups + grp; r < R; r += gridDim.x * groups) {
        int s = 0;
        while (off[s + 1] <= r) ++s;
        const size_t row = (size_t)s * p.m_max + (r - off[s]);
        const uint4* src = reinterpret_cast<const uint4*>(rx + row * H);
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
        for (int i = gt; i < p.meta; i += gsz) meta_rows[(size_t)r * p.meta + i] = __ldcg(rm + row * p.meta + i);
    }
}

// Gate-weighted identity expert stage (region mode): y[s][j] = (sum of the row's local gate
// weights) * x[s][j] for every received row — the stand-in for the expert FFN (a library GEMM,
// out of scope) in benches and whole-layer graphs.  Reads this step's region through the device
// epoch, so a captured graph replays it on either parity.  One warp per row.
static __global__ void __launch_bounds__(256) moe_expert_identity_kernel(const __grid_constant__ MoePeers p,
                                                                         __nv_bfloat16* __restrict__ y_region) {
    pdl_trigger();  // MoE launches are PDL-chained (capi_moe.cu)
    pdl_wait();
    const uint32_t ep = *p.epoch;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int R = p.offs[p.W];
    const __nv_bfloat16* rx = rx_x(p, p.self, ep);
    const int32_t* rm = rx_meta(p, p.self, ep);
    const int nvec = p.H / 8;
    for (int r = warp; r < R; r += nwarps) {
        int s = 0;
        while (p.offs[s + 1] <= r) ++s;
        const size_t row = (size_t)s * p.m_max + (r - p.offs[s]);
        const int32_t* meta = rm + row * p.meta;
        const int n = __ldcg(meta + 1);
        float wsum = 0.f;
        for (int i = 0; i < n; ++i) wsum += __int_as_float(__ldcg(meta + 3 + 2 * i));
        const uint4* src = reinterpret_cast<const uint4*>(rx + row * p.H);
        uint4* dst = reinterpret_cast<uint4*>(y_region + row * p.H);
        for (int i = lane; i < nvec; i += 32) {
            uint4 v = __ldcg(src + i);
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 f = __bfloat1622float2(h[k]);
                h[k] = __floats2bfloat162_rn(f.x * wsum, f.y * wsum);
            }
            dst[i] = v;
        }
    }
}

// K5b body: returns received rows (flattened source-major) to their homes, one warp per row.
// y_rows: compact [R][H] (row = offs[s] + j) or region [W][m_max][H] (row = s * m_max + j).
__device__ __forceinline__ void combine_put_body(const MoePeers& p, const __nv_bfloat16* __restrict__ y_rows,
                                                 int region) {
    __shared__ int32_t s_off[PL_MAXW + 1], s_sent[PL_MAXW];
    const uint32_t ep = *p.epoch;
    const int W = p.W, H = p.H, tid = threadIdx.x;
    if (tid <= W) s_off[tid] = p.offs[tid];
    if (tid < PL_MAXW) s_sent[tid] = 0;
    __syncthreads();
    const int R = s_off[W];
    const int nvec = H / 8;
    const int32_t* rm = rx_meta(p, p.self, ep);
#if MOE_K5B_WARP
    // one warp per received row, 8 vectors per lane in flight
    constexpr int VPL = 8;
    const int lane = tid & 31;
    const int nwarps = gridDim.x * (MOE_THREADS / 32);
    for (int r = blockIdx.x * (MOE_THREADS / 32) + (tid >> 5); r < R; r += nwarps) {
        int s = 0;
        while (s_off[s + 1] <= r) ++s;
        const int j = r - s_off[s];
        const int t = __ldcg(rm + ((size_t)s * p.m_max + j) * p.meta);
        const uint4* src =
            reinterpret_cast<const uint4*>(y_rows + (size_t)(region ? s * p.m_max + j : r) * H);
        uint4* dst = reinterpret_cast<uint4*>(cb_y(p, s, ep) + ((size_t)t * W + p.self) * H);
        for (int v0 = lane; v0 < nvec; v0 += VPL * 32) {
            uint4 v[VPL];
#pragma unroll
            for (int u = 0; u < VPL; ++u)
                if (v0 + u * 32 < nvec) v[u] = __ldg(src + v0 + u * 32);
#pragma unroll
            for (int u = 0; u < VPL; ++u)
                if (v0 + u * 32 < nvec) dst[v0 + u * 32] = v[u];
        }
        if (lane == 0) atomicAdd(&s_sent[s], 1);
    }
#else
    constexpr int VPT = 4;
    for (int r = blockIdx.x; r < R; r += gridDim.x) {
        int s = 0;
        while (s_off[s + 1] <= r) ++s;
        const int j = r - s_off[s];
        const int t = __ldcg(rm + ((size_t)s * p.m_max + j) * p.meta);
        const uint4* src =
            reinterpret_cast<const uint4*>(y_rows + (size_t)(region ? s * p.m_max + j : r) * H);
        uint4* dst = reinterpret_cast<uint4*>(cb_y(p, s, ep) + ((size_t)t * W + p.self) * H);
        for (int v0 = tid; v0 < nvec; v0 += VPT * MOE_THREADS) {
            uint4 v[VPT];
#pragma unroll
            for (int u = 0; u < VPT; ++u)
                if (v0 + u * MOE_THREADS < nvec) v[u] = __ldg(src + v0 + u * MOE_THREADS);
#pragma unroll
            for (int u = 0; u < VPT; ++u)
                if (v0 + u * MOE_THREADS < nvec) dst[v0 + u * MOE_THREADS] = v[u];
        }
        if (tid == 0) ++s_sent[s];
    }
#endif
    __syncthreads();
#if MOE_SINGLE_RELEASE
    if (tid == 0) {
        int old;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(p.exit_ticket) : "memory");
        if (old == static_cast<int>(gridDim.x) - 1) {
            *p.exit_ticket = 0;
            asm volatile("fence.acq_rel.sys;" ::: "memory");
            for (int d = 0; d < W; ++d)
                if (s_off[d + 1] > s_off[d])
                    asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(cb_arr(p, d, ep) + p.self),
                                 "r"(s_off[d + 1] - s_off[d]) : "memory");
        }
    }
#else
    if (tid < W && s_sent[tid]) red_release_sys_add(cb_arr(p, tid, ep) + p.self, s_sent[tid]);
#endif
}

// K5b: one launch of the body.
static __global__ void __launch_bounds__(MOE_THREADS) moe_combine_put_kernel(const __grid_constant__ MoePeers p,
                                                                             const __nv_bfloat16* __restrict__ y_rows,
                                                                             int region) {
    pdl_trigger();  // MoE launches are PDL-chained (capi_moe.cu)
    pdl_wait();
    combine_put_body(p, y_rows, region);
}

// K5c's per-(token, 4-column group) reduction: every routed rank's bf16 partial, ascending rank
// (= ascending expert) order, fp32; the W loads are in flight together.
__device__ __forceinline__ void reduce_token_cols(const MoePeers& p, int t, int q, uint32_t dm, uint32_t ep,
                                                  float* __restrict__ out) {
    const int W = p.W, H = p.H;
    const __nv_bfloat16* cy = cb_y(p, p.self, ep);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    uint2 v[PL_MAXW];
#pragma unroll 8
    for (int d = 0; d < W; ++d)
        if ((dm >> d) & 1u)
            v[d] = __ldcg(reinterpret_cast<const uint2*>(cy + ((size_t)t * W + d) * H) + q);
#pragma unroll 8
    for (int d = 0; d < W; ++d) {
        if (!((dm >> d) & 1u)) continue;
        const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v[d].x));
        const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v[d].y));
        a0 += lo.x;
        a1 += lo.y;
        a2 += hi.x;
        a3 += hi.y;
    }
    reinterpret_cast<float4*>(out + (size_t)t * H)[q] = make_float4(a0, a1, a2, a3);
}

// K5c: at home, sum the partials of every destination rank in ascending order.  CTA (token t,
// hidden chunk); each thread owns 4 consecutive columns.
static __global__ void __launch_bounds__(256) moe_combine_reduce_kernel(const __grid_constant__ MoePeers p,
                                                                        const int32_t* __restrict__ m_count,
                                                                        float* __restrict__ out) {
    pdl_trigger();  // MoE launches are PDL-chained (capi_moe.cu)
    pdl_wait();
    const int t = blockIdx.x;
    if (t >= *m_count) return;
    const uint32_t ep = *p.epoch;
    const int W = p.W, H = p.H;
    // the token's destination set (this instance's own K4 layout) is read before the flag wait
    uint32_t dm = 0;
#pragma unroll 8
    for (int d = 0; d < W; ++d) dm |= (p.slot_tbl[t * W + d] >= 0 ? 1u : 0u) << d;
    if (threadIdx.x < W)
        wait_flag(cb_arr(p, p.self, ep) + threadIdx.x, p.cb_target[(ep & 1) * W + threadIdx.x], p.wc,
                  (SITE_MOE_CB << 24) | (threadIdx.x << 16) | (t & 0xffff), true);
    __syncthreads();
    const int q = blockIdx.y * blockDim.x + threadIdx.x;  // 4-column group
    if (4 * q >= H) return;
    reduce_token_cols(p, t, q, dm, ep, out);
}

// Fused combine (multi-process / multi-GPU only): K5b's puts, then K5c's reduction of this
// instance's tokens, in one grid.  The reduction waits for every rank's rows, this grid's own
// included (its last CTA publishes them, single release); the CTAs are co-resident (grid =
// SMs) and the peers run concurrently on their own GPUs.  Instances sharing one GPU in one
// process keep the two launches: a spinning reduction would hold the SMs a peer's puts need.
static __global__ void __launch_bounds__(MOE_THREADS) moe_combine_fused_kernel(const __grid_constant__ MoePeers p,
                                                                               const __nv_bfloat16* __restrict__ y_region,
                                                                               const int32_t* __restrict__ m_count,
                                                                               float* __restrict__ out) {
    pdl_trigger();  // MoE launches are PDL-chained (capi_moe.cu)
    pdl_wait();
    combine_put_body(p, y_region, 1);
    const uint32_t ep = *p.epoch;
    const int W = p.W, H = p.H, M = *m_count;
    if (static_cast<int>(blockIdx.x) >= M) return;
    if (threadIdx.x < W)
        wait_flag(cb_arr(p, p.self, ep) + threadIdx.x, p.cb_target[(ep & 1) * W + threadIdx.x], p.wc,
                  (SITE_MOE_CB << 24) | (threadIdx.x << 16) | (blockIdx.x & 0xffff), true);
    __syncthreads();
    for (int t = blockIdx.x; t < M; t += gridDim.x) {
        uint32_t dm = 0;
#pragma unroll 8
        for (int d = 0; d < W; ++d) dm |= (p.slot_tbl[t * W + d] >= 0 ? 1u : 0u) << d;
        for (int q = threadIdx.x; 4 * q < H; q += blockDim.x) reduce_token_cols(p, t, q, dm, ep, out);
    }
}

}  // namespace dcp
