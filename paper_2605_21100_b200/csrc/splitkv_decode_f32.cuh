// SPDX-License-Identifier: Apache-2.0
//
// K1-f32: split-KV paged decode attention in fp32 — the precision of the
// reference's production path (shard_attention<float> / lse_merge<float>,
// attn_merge.hpp:53-100; explicit float instantiation attn_merge.cpp:64-77;
// SPEC.md:380 fp32 rel <= 1e-5).  BASELINE configs[0] (cfg1) runs here.
//
// Semantics per (shard r, q-head h) are those of K1 (splitkv_decode.cuh):
//   s_j = scale * <q, k_j>,  O = softmax(s) V (normalised),  lse = max + ln sum exp(s - max)
// computed with fp32 FMAs and expf/logf (no bf16 rounding of P, no exp2 rescaling).
//
// Design: the same persistent stream-K split of the flattened page sequence as
// K1 (every CTA streams an equal page range whatever the length skew), the same
// (acc, max, sum) partial slots and last-arriver merge (K9), and the same routed
// epilogue (Res-route put + flag, exchange.cuh).  The inner loop is CUDA-core
// fp32: one warp per kv-head, each lane owns 4 of the 128 head dims (one
// 16-byte load per K / V row and lane, 512-byte coalesced rows); TOK tokens are
// in flight per warp, their G x TOK dot products reduced with one butterfly per
// token; online softmax per q-head in registers.  fp32 KV is 2x the bytes of
// bf16 and arithmetic intensity is ~0.5 flop/B per q-head: HBM-bound.
#pragma once

#include <cstdint>

#include "exchange.cuh"
#include "ptx.cuh"

namespace dcp {

struct AttnF32Params {
    const float* q;              // [R][HQ][128] (local mode)
    const float* kv;             // [frames][2][HKV][page][128]
    const int32_t* block_table;  // [P]
    const int32_t* cu_pages;     // [R+1]
    const int64_t* shard_len;    // [R]
    const uint8_t* page_fill;    // [P] or nullptr
    float* out;                  // [R][HQ][128]
    float* lse;                  // [R][HQ]
    float* ws_acc;               // [2*grid][HQ][128]
    float* ws_ml;                // [2*grid][HQ][2]
    int32_t* counters;           // [R]
    int32_t num_shards;
    int32_t hkv;
    int32_t page;
    float scale;
    const XchgPeers* xp;         // routed mode (see AttnParams)
    const int32_t* n_mrow;
    const int32_t* n_moe;
    const int32_t* num_shards_ptr;
};

constexpr int F32_D = 128;

// Stream-K helpers shared with K1.
__device__ __forceinline__ int f32_cta_of_page(int64_t p, int64_t P, int64_t grid) {
    return static_cast<int>(udiv64((p + 1) * grid + P - 1, P) - 1);
}
__device__ __forceinline__ bool f32_cta_nonempty(int64_t k, int64_t P, int64_t grid) {
    return P >= grid || udiv64(k * P, grid) < udiv64((k + 1) * P, grid);
}

template <class P>
__device__ __forceinline__ float* f32_row_out(const P& p, int r, int HQ, uint32_t ep) {
    if (!p.xp) return p.out + (size_t)r * HQ * F32_D;
    const XchgPeers& x = *p.xp;
    return xres_o(x, p.n_moe[r], ep) + ((size_t)p.n_mrow[r] * x.W + x.self) * HQ * F32_D;
}
template <class P>
__device__ __forceinline__ float* f32_row_lse(const P& p, int r, int HQ, uint32_t ep) {
    if (!p.xp) return p.lse + (size_t)r * HQ;
    const XchgPeers& x = *p.xp;
    return xres_lse(x, p.n_moe[r], ep) + ((size_t)p.n_mrow[r] * x.W + x.self) * HQ;
}
template <class P>
__device__ __forceinline__ void f32_publish_row(const P& p, int r, uint32_t ep) {
    const XchgPeers& x = *p.xp;
    st_release_sys(xres_flag(x, p.n_moe[r], ep) + (size_t)p.n_mrow[r] * x.W + x.self, ep);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block = hkv (<= 8) warps, one per kv-head; grid = persistent, any size.
template <int G>
__global__ void __launch_bounds__(256) splitkv_decode_f32_kernel(const AttnF32Params p) {
    constexpr int TOK = 8;  // tokens in flight per warp
    __shared__ int s_last;
    const int h = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int HKV = p.hkv, HQ = HKV * G, PG = p.page;
    const int nthreads = HKV * 32;
    const int R = p.num_shards_ptr ? *p.num_shards_ptr : p.num_shards;
    const uint32_t ep = p.xp ? *p.xp->epoch : 0u;
    const float* qbase = p.xp ? reinterpret_cast<const float*>(xq_recv(*p.xp, p.xp->self, ep)) : p.q;
    const uint32_t* qflag = p.xp ? xq_flag(*p.xp, p.xp->self, ep) : nullptr;
    const int64_t P = p.cu_pages[R];
    const int64_t grid = gridDim.x;
    const int cta = blockIdx.x;
    const int p_begin = static_cast<int>(udiv64(cta * P, grid));
    const int p_end = static_cast<int>(udiv64((cta + 1) * P, grid));

    // zero-token shards: O = 0, LSE = -inf
    for (int r = cta; r < R; r += gridDim.x) {
        if (p.cu_pages[r + 1] == p.cu_pages[r]) {
            float* ob = f32_row_out(p, r, HQ, ep);
            float* lb = f32_row_lse(p, r, HQ, ep);
            for (int g = 0; g < G; ++g) {
                reinterpret_cast<float4*>(ob + (h * G + g) * F32_D)[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (lane == 0) lb[h * G + g] = -INFINITY;
            }
            if (p.xp) {
                named_bar_sync(1, nthreads);
                if (threadIdx.x == 0) f32_publish_row(p, r, ep);
            }
        }
    }
    if (p_begin >= p_end) return;

    int r;
    {
        int lo = 0, hi = R;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (p.cu_pages[mid] <= p_begin) lo = mid; else hi = mid - 1;
        }
        r = lo;
    }
    const size_t head_stride = (size_t)PG * F32_D;       // one (part, head) block of a frame
    const size_t frame_stride = 2 * (size_t)HKV * head_stride;
    int pg = p_begin;
    while (pg < p_end) {
        while (p.cu_pages[r + 1] <= pg) ++r;
        const int r_first = p.cu_pages[r], r_last = p.cu_pages[r + 1];
        const int seg_begin = pg, seg_end = min(r_last, p_end);
        const int64_t len = p.shard_len[r];
        if (qflag) {
            if (lane == 0) wait_flag(qflag + r, ep, p.xp->wc, (SITE_K1_Q << 24) | (r & 0xffff));
            __syncwarp();
        }
        float4 q[G];
#pragma unroll
        for (int g = 0; g < G; ++g)
            q[g] = __ldcg(reinterpret_cast<const float4*>(qbase + ((size_t)r * HQ + h * G + g) * F32_D) + lane);
        float m[G], l[G];
        float4 acc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            m[g] = -INFINITY;
            l[g] = 0.f;
            acc[g] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (; pg < seg_end; ++pg) {
            const int f = __ldg(p.block_table + pg);
            int fill;
            if (p.page_fill) {
                fill = __ldg(p.page_fill + pg);
            } else {
                const int64_t rem = len - static_cast<int64_t>(pg - r_first) * PG;
                fill = rem < PG ? static_cast<int>(rem) : PG;
            }
            const float* kb = p.kv + (size_t)f * frame_stride + (size_t)h * head_stride;
            const float* vb = kb + (size_t)HKV * head_stride;
            for (int t0 = 0; t0 < fill; t0 += TOK) {
                const int nt = min(TOK, fill - t0);
                float4 kr[TOK], vr[TOK];
#pragma unroll
                for (int u = 0; u < TOK; ++u) {
                    kr[u] = vr[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (u < nt) {
                        kr[u] = __ldcs(reinterpret_cast<const float4*>(kb + (size_t)(t0 + u) * F32_D) + lane);
                        vr[u] = __ldcs(reinterpret_cast<const float4*>(vb + (size_t)(t0 + u) * F32_D) + lane);
                    }
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    float s[TOK];
                    float mx = m[g];
#pragma unroll
                    for (int u = 0; u < TOK; ++u) {
                        float d = q[g].x * kr[u].x;
                        d = fmaf(q[g].y, kr[u].y, d);
                        d = fmaf(q[g].z, kr[u].z, d);
                        d = fmaf(q[g].w, kr[u].w, d);
                        d = warp_sum(d);
                        s[u] = u < nt ? p.scale * d : -INFINITY;
                        mx = fmaxf(mx, s[u]);
                    }
                    const float alpha = expf(m[g] - mx);  // m = -inf on the first tokens: 0
                    float4 a = acc[g];
                    a.x *= alpha;
                    a.y *= alpha;
                    a.z *= alpha;
                    a.w *= alpha;
                    float ls = l[g] * alpha;
#pragma unroll
                    for (int u = 0; u < TOK; ++u) {
                        if (u < nt) {
                            const float w = expf(s[u] - mx);
                            ls += w;
                            a.x = fmaf(w, vr[u].x, a.x);
                            a.y = fmaf(w, vr[u].y, a.y);
                            a.z = fmaf(w, vr[u].z, a.z);
                            a.w = fmaf(w, vr[u].w, a.w);
                        }
                    }
                    acc[g] = a;
                    l[g] = ls;
                    m[g] = mx;
                }
            }
        }
        const bool complete = (seg_begin == r_first) && (seg_end == r_last);
        if (complete) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int qh = h * G + g;
                const float inv = 1.f / l[g];
                reinterpret_cast<float4*>(f32_row_out(p, r, HQ, ep) + qh * F32_D)[lane] =
                    make_float4(acc[g].x * inv, acc[g].y * inv, acc[g].z * inv, acc[g].w * inv);
                if (lane == 0) f32_row_lse(p, r, HQ, ep)[qh] = m[g] + logf(l[g]);
            }
            if (p.xp) {
                named_bar_sync(1, nthreads);
                if (threadIdx.x == 0) f32_publish_row(p, r, ep);
            }
        } else {
            const int slot = 2 * cta + (seg_begin == p_begin ? 0 : 1);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int qh = h * G + g;
                __stcg(reinterpret_cast<float4*>(p.ws_acc + ((size_t)slot * HQ + qh) * F32_D) + lane, acc[g]);
                if (lane == 0)
                    __stcg(reinterpret_cast<float2*>(p.ws_ml) + ((size_t)slot * HQ + qh), make_float2(m[g], l[g]));
            }
            named_bar_sync(1, nthreads);  // the partial stores happen-before thread 0's release
            if (threadIdx.x == 0) {
                const int a = f32_cta_of_page(r_first, P, grid), b = f32_cta_of_page(r_last - 1, P, grid);
                const int nparts = P < grid ? r_last - r_first : b - a + 1;  // P < grid: one page per CTA
                s_last = atom_add_acq_rel_gpu(p.counters + r, 1) == nparts - 1;
            }
            named_bar_sync(1, nthreads);
            if (s_last) {
                const int a = f32_cta_of_page(r_first, P, grid), b = f32_cta_of_page(r_last - 1, P, grid);
                auto slot_of = [&](int k) {
                    return (k == a && r_first != static_cast<int>(k * P / grid)) ? 2 * k + 1 : 2 * k;
                };
                // lse_merge over the parts in page order (attn_merge.hpp:86-100), fp32, expf
                for (int g = 0; g < G; ++g) {
                    const int qh = h * G + g;
                    float mmax = -INFINITY;
                    for (int k = a; k <= b; ++k)
                        if (f32_cta_nonempty(k, P, grid))
                            mmax = fmaxf(mmax, __ldcg(reinterpret_cast<const float2*>(p.ws_ml) +
                                                      ((size_t)slot_of(k) * HQ + qh)).x);
                    float den = 0.f;
                    float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
                    for (int k = a; k <= b; ++k) {
                        if (!f32_cta_nonempty(k, P, grid)) continue;
                        const int sl = slot_of(k);
                        const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.ws_ml) + ((size_t)sl * HQ + qh));
                        const float w = expf(ml.x - mmax);
                        den = fmaf(w, ml.y, den);
                        const float4 v = __ldcg(reinterpret_cast<const float4*>(p.ws_acc + ((size_t)sl * HQ + qh) * F32_D) + lane);
                        num.x = fmaf(w, v.x, num.x);
                        num.y = fmaf(w, v.y, num.y);
                        num.z = fmaf(w, v.z, num.z);
                        num.w = fmaf(w, v.w, num.w);
                    }
                    const float inv = 1.f / den;
                    reinterpret_cast<float4*>(f32_row_out(p, r, HQ, ep) + qh * F32_D)[lane] =
                        make_float4(num.x * inv, num.y * inv, num.z * inv, num.w * inv);
                    if (lane == 0) f32_row_lse(p, r, HQ, ep)[qh] = mmax + logf(den);
                }
                if (threadIdx.x == 0) p.counters[r] = 0;
                if (p.xp) {
                    named_bar_sync(2, nthreads);
                    if (threadIdx.x == 0) f32_publish_row(p, r, ep);
                }
            }
        }
        ++r;
    }
}

}  // namespace dcp
