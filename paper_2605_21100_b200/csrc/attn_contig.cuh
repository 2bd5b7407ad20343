// SPDX-License-Identifier: Apache-2.0
//
// K1f / K9f: fp32 / fp64 attention over contiguous spans — the reference's
// math API on device:
//   shard_attention<T>  attn_merge.hpp:53-82  (one item = one query x one shard)
//   lse_merge<T>        attn_merge.hpp:86-100 (one group = one partial list)
// Used by the dcpsim C++ drop-in (include/dcpsim/attn_merge.hpp) and for the
// fp32 configuration (BASELINE configs[0]); the bf16 paged decode path is K1.
// CUDA cores: 4 warps per item split the keys, lanes own head-dim slices, a
// warp all-reduce forms each score, per-warp online softmax, then a
// shared-memory merge of the 4 warp states (the same LSE identity).
#pragma once

#include <cstdint>

namespace dcp {

template <typename T>
__device__ __forceinline__ T dexp(T x);
template <>
__device__ __forceinline__ float dexp<float>(float x) { return expf(x); }
template <>
__device__ __forceinline__ double dexp<double>(double x) { return exp(x); }
template <typename T>
__device__ __forceinline__ T dlog(T x);
template <>
__device__ __forceinline__ float dlog<float>(float x) { return logf(x); }
template <>
__device__ __forceinline__ double dlog<double>(double x) { return log(x); }

constexpr int CONTIG_MAXD = 256;

template <typename T>
__global__ void __launch_bounds__(128) shard_attn_contig_kernel(int d, T scale, const T* __restrict__ q,
                                                                const T* __restrict__ keys,
                                                                const T* __restrict__ values,
                                                                const int64_t* __restrict__ q_off,
                                                                const int64_t* __restrict__ kv_off,
                                                                const int64_t* __restrict__ len,
                                                                T* __restrict__ out, T* __restrict__ lse) {
    constexpr int NW = 4;
    constexpr int PER = CONTIG_MAXD / 32;
    __shared__ T s_m[NW], s_l[NW];
    __shared__ T s_acc[NW][CONTIG_MAXD];
    const int item = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const T* qi = q + q_off[item];
    const T* K = keys + kv_off[item];
    const T* V = values + kv_off[item];
    const int64_t L = len[item];
    T qv[PER], acc[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int dd = lane + 32 * j;
        qv[j] = dd < d ? qi[dd] : T(0);
        acc[j] = T(0);
    }
    T m = -INFINITY, l = T(0);
    for (int64_t t = warp; t < L; t += NW) {
        const T* kt = K + t * d;
        const T* vt = V + t * d;
        T part = T(0);
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int dd = lane + 32 * j;
            if (dd < d) part += kt[dd] * qv[j];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        const T s = part * scale;
        if (s > m) {
            const T shrink = dexp<T>(m - s);
            l *= shrink;
#pragma unroll
            for (int j = 0; j < PER; ++j) acc[j] *= shrink;
            m = s;
        }
        const T w = dexp<T>(s - m);
        l += w;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int dd = lane + 32 * j;
            if (dd < d) acc[j] += w * vt[dd];
        }
    }
    if (lane == 0) {
        s_m[warp] = m;
        s_l[warp] = l;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int dd = lane + 32 * j;
        if (dd < d) s_acc[warp][dd] = acc[j];
    }
    __syncthreads();
    T M = -INFINITY;
    for (int w = 0; w < NW; ++w) M = s_m[w] > M ? s_m[w] : M;
    T den = T(0);
    T wt[NW];
    for (int w = 0; w < NW; ++w) {
        wt[w] = s_m[w] == -INFINITY ? T(0) : dexp<T>(s_m[w] - M);
        den += wt[w] * s_l[w];
    }
    for (int dd = threadIdx.x; dd < d; dd += blockDim.x) {
        T num = T(0);
        for (int w = 0; w < NW; ++w) num += wt[w] * s_acc[w][dd];
        out[(int64_t)item * d + dd] = L > 0 ? num / den : T(0);
    }
    if (threadIdx.x == 0) lse[item] = L > 0 ? M + dlog<T>(den) : T(-INFINITY);
}

// lse_merge over groups: group g = partials [g_off[g], g_off[g+1]) in list order.
template <typename T>
__global__ void __launch_bounds__(128) lse_merge_contig_kernel(int d, const int64_t* __restrict__ g_off,
                                                               const T* __restrict__ outs,
                                                               const T* __restrict__ lses,
                                                               T* __restrict__ merged, T* __restrict__ merged_lse) {
    const int g = blockIdx.x;
    const int64_t a = g_off[g], b = g_off[g + 1];
    T M = -INFINITY;
    for (int64_t i = a; i < b; ++i) M = lses[i] > M ? lses[i] : M;
    T ws = T(0);
    for (int64_t i = a; i < b; ++i) ws += lses[i] == -INFINITY ? T(0) : dexp<T>(lses[i] - M);
    for (int dd = threadIdx.x; dd < d; dd += blockDim.x) {
        T acc = T(0);
        for (int64_t i = a; i < b; ++i) {
            const T w = lses[i] == -INFINITY ? T(0) : dexp<T>(lses[i] - M);
            acc += w * outs[i * d + dd];
        }
        merged[(int64_t)g * d + dd] = acc / ws;
    }
    if (threadIdx.x == 0 && merged_lse) merged_lse[g] = M + dlog<T>(ws);
}

}  // namespace dcp
