// SPDX-License-Identifier: Apache-2.0
// K2 / K3 kernels (see exchange.cuh for the protocol).  Included by capi_xchg.cu only.
#pragma once
#include "exchange.cuh"

namespace dcp {

static __global__ void epoch_bump_kernel(uint32_t* epoch) { *epoch += 1; }

// K2: grid = m_max (graph-stable), block = 128.  q_local: [m_max][hq][d] bf16
// in M-row order; m_nrow: [M][W] destination rows (-1 = not in P_r).
static __global__ void __launch_bounds__(128) q_route_put_kernel(const XchgPeers* __restrict__ xp,
                                                          const __nv_bfloat16* __restrict__ q_local,
                                                          const int32_t* __restrict__ m_count,
                                                          const int32_t* __restrict__ m_nrow) {
    const int r = blockIdx.x;
    const XchgPeers& x = *xp;
    if (r >= m_count[x.self]) return;
    const uint32_t ep = *x.epoch;
    const int W = x.W;
    const int vecs = x.hq * x.d / 8;  // 16-byte vectors per query row
    const uint4* src = reinterpret_cast<const uint4*>(q_local + (size_t)r * x.hq * x.d);
    for (int s = 0; s < W; ++s) {
        const int row = m_nrow[(size_t)r * W + s];
        if (row < 0) continue;
        uint4* dst = reinterpret_cast<uint4*>(x.qrecv[s] + (size_t)row * x.hq * x.d);
        for (int i = threadIdx.x; i < vecs; i += blockDim.x) dst[i] = __ldg(src + i);
        __syncthreads();
        if (threadIdx.x == 0) st_release_sys(x.qflag[s] + row, ep);
    }
}

// K3 merge: grid = m_max, block = 128.  m_k / m_kv: P_r of each M row in
// kv_binding order.  out: [m_max][hq][d] fp32, out_lse: [m_max][hq].
static __global__ void __launch_bounds__(128) lse_merge_kernel(const XchgPeers* __restrict__ xp,
                                                        const int32_t* __restrict__ m_count,
                                                        const int32_t* __restrict__ m_k,
                                                        const int32_t* __restrict__ m_kv,
                                                        float* __restrict__ out,
                                                        float* __restrict__ out_lse) {
    const int r = blockIdx.x;
    const XchgPeers& x = *xp;
    if (r >= m_count[x.self]) return;
    const uint32_t ep = *x.epoch;
    const int W = x.W, hq = x.hq, d = x.d;
    const int k = m_k[r];
    __shared__ int32_t parts[PL_MAXK];
    if (threadIdx.x < k) {
        const int s = m_kv[(size_t)r * PL_MAXK + threadIdx.x];
        parts[threadIdx.x] = s;
        wait_flag(x.res_flag[x.self] + (size_t)r * W + s, ep);
    }
    __syncthreads();
    const float* po = x.res_o[x.self] + (size_t)r * W * hq * d;
    const float* pl = x.res_lse[x.self] + (size_t)r * W * hq;
    const float L2E = 1.4426950408889634f;
    const int quarters = d / 32;  // 32 floats per work item
    for (int w = threadIdx.x; w < hq * quarters; w += blockDim.x) {
        const int h = w / quarters, q0 = (w % quarters) * 32;
        float mx = -INFINITY;
        for (int i = 0; i < k; ++i) mx = fmaxf(mx, __ldcg(pl + (size_t)parts[i] * hq + h));
        float acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.f;
        float den = 0.f;
        for (int i = 0; i < k; ++i) {
            const int s = parts[i];
            const float l = __ldcg(pl + (size_t)s * hq + h);
            const float wgt = l == -INFINITY ? 0.f : exp2f((l - mx) * L2E);
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
}

}  // namespace dcp
