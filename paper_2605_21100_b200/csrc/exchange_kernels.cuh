// SPDX-License-Identifier: Apache-2.0
// K2 / K3 kernels (see exchange.cuh for the protocol).  Included by capi_xchg.cu only.
#pragma once
#include "exchange.cuh"

namespace dcp {

// begin_step: the step fence of exchange.cuh, then the epoch bump.  One warp.
static __global__ void __launch_bounds__(32) xchg_begin_step_kernel(const __grid_constant__ XchgPeers x) {
    step_fence(x.epoch, [&](int s) { return xdone(x, s); }, x.W, x.self, x.wc);
}

// K2: grid = m_max (graph-stable), block = 128.  q_local: [m_max][hq][q_dim] x q_bytes
// in M-row order; m_nrow: [M][W] destination rows (-1 = not in P_r).  The payload is
// moved as 16-byte vectors whatever its element type (bf16 Q, fp32 Q, MLA's 576-wide Q).
static __global__ void __launch_bounds__(128) q_route_put_kernel(const __grid_constant__ XchgPeers x,
                                                                 const void* __restrict__ q_local,
                                                                 const int32_t* __restrict__ m_count,
                                                                 const int32_t* __restrict__ m_nrow) {
    const int M = m_count[x.self];
    const uint32_t ep = *x.epoch;
    const int W = x.W;
    const size_t row_bytes = (size_t)x.hq * x.q_dim * x.q_bytes;
    const int vecs = static_cast<int>(row_bytes / 16);
    constexpr int U = 4;
    // grid-stride over the M rows: any grid (an M-bucket's, or fewer) covers every row
    for (int r = blockIdx.x; r < M; r += gridDim.x) {
        const uint4* src = reinterpret_cast<const uint4*>(static_cast<const char*>(q_local) + r * row_bytes);
        for (int s = 0; s < W; ++s) {
            const int row = m_nrow[(size_t)r * W + s];
            if (row < 0) continue;
            uint4* dst = reinterpret_cast<uint4*>(xq_recv(x, s, ep) + row * row_bytes);
            for (int b = threadIdx.x; b < vecs; b += U * blockDim.x) {
                uint4 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (b + u * blockDim.x < vecs) v[u] = __ldg(src + b + u * blockDim.x);
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (b + u * blockDim.x < vecs) dst[b + u * blockDim.x] = v[u];
            }
            __syncthreads();
            if (threadIdx.x == 0) st_release_sys(xq_flag(x, s, ep) + row, ep);
        }
    }
}

// K3 merge: grid = m_max, block = 128.  m_k / m_kv: P_r of each M row in kv_binding
// order.  out: [m_max][hq][o_dim] fp32, out_lse: [m_max][hq].  Weights follow lse_merge
// (attn_merge.hpp:86-100): w_k = exp(lse_k - max lse), out = sum w_k o_k / sum w_k, folded
// in kv_binding order; an empty shard (lse = -inf) has weight 0.
static __global__ void __launch_bounds__(128) lse_merge_kernel(const __grid_constant__ XchgPeers x,
                                                               const int32_t* __restrict__ m_count,
                                                               const int32_t* __restrict__ m_k,
                                                               const int32_t* __restrict__ m_kv,
                                                               float* __restrict__ out,
                                                               float* __restrict__ out_lse) {
    const int M = m_count[x.self];
    const uint32_t ep = *x.epoch;
    const int W = x.W, hq = x.hq, d = x.o_dim;
    __shared__ int32_t parts[PL_MAXK];
    for (int r = blockIdx.x; r < M; r += gridDim.x) {  // grid-stride: any grid covers every row
        const int k = m_k[r];
        if (threadIdx.x < k) {
            const int s = m_kv[(size_t)r * PL_MAXK + threadIdx.x];
            parts[threadIdx.x] = s;
            wait_flag(xres_flag(x, x.self, ep) + (size_t)r * W + s, ep, x.wc,
                      (SITE_K3_RES << 24) | (s << 16) | (r & 0xffff));
        }
        __syncthreads();
        const float* po = xres_o(x, x.self, ep) + (size_t)r * W * hq * d;
        const float* pl = xres_lse(x, x.self, ep) + (size_t)r * W * hq;
        const int chunks = d / 32;  // 32 floats per work item
        for (int w = threadIdx.x; w < hq * chunks; w += blockDim.x) {
            const int h = w / chunks, q0 = (w % chunks) * 32;
            float mx = -INFINITY;
            for (int i = 0; i < k; ++i) mx = fmaxf(mx, __ldcg(pl + (size_t)parts[i] * hq + h));
            float acc[32];
    #pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] = 0.f;
            float den = 0.f;
            for (int i = 0; i < k; ++i) {
                const int s = parts[i];
                const float l = __ldcg(pl + (size_t)s * hq + h);
                const float wgt = l == -INFINITY ? 0.f : expf(l - mx);
                den += wgt;
                const float4* v = reinterpret_cast<const float4*>(po + ((size_t)s * hq + h) * d + q0);
    #pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 t = __ldcg(v + j);
                    acc[4 * j] += wgt * t.x;
                    acc[4 * j + 1] += wgt * t.y;
                    acc[4 * j + 2] += wgt * t.z;
                    acc[4 * j + 3] += wgt * t.w;
                }
            }
            const float inv = 1.f / den;
            float4* o = reinterpret_cast<float4*>(out + ((size_t)r * hq + h) * d + q0);
    #pragma unroll
            for (int j = 0; j < 8; ++j)
                o[j] = make_float4(acc[4 * j] * inv, acc[4 * j + 1] * inv, acc[4 * j + 2] * inv, acc[4 * j + 3] * inv);
            if (q0 == 0) out_lse[(size_t)r * hq + h] = mx + logf(den);
        }
        __syncthreads();  // parts[] is rewritten by the next row
    }
}

}  // namespace dcp
