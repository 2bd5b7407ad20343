// SPDX-License-Identifier: Apache-2.0
//
// K2 / K3: the routing-based communication backend of the DCP decode step
// (north_star subsystem 2; Fig. 7 phases 1 and 3-4).
//
//   K2  q_route_put     at the MoE binding m: for every M row r and every
//                       s in P_r, store Q_r into s's query receive slot (row of
//                       r in s's N list) with st.global — a peer-mapped NVLink
//                       address when s is another GPU — then publish a
//                       per-row arrival flag (st.release.sys = epoch).
//   K1  (epilogue)      each KV-binding instance s stores the partial O and LSE
//                       of row r straight into m_r's result pool slot
//                       [mrow(r)][s] and publishes a per-(row, s) flag — the
//                       Res-route put is fused into the attention kernel.
//   K3  lse_merge       at m: wait for the |P_r| flags, merge in kv_binding
//                       order with the math of lse_merge (attn_merge.hpp:86-100);
//                       zero-token shards carry LSE = -inf (weight 0), which is
//                       how the reference's "drop empty partials" (attn_merge.cpp:41-44)
//                       is expressed without a data-dependent list.
//
// Flags carry an epoch (bumped once per step on every instance) so CUDA-graph
// replay needs no flag reset.  Self routes (s == m) use the same path on
// local memory.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>

#include "limits.cuh"

namespace dcp {

struct XchgPeers {
    int32_t W, self, hq, d, n_max, m_max;
    uint32_t* epoch;                  // local, bumped per step
    __nv_bfloat16* qrecv[PL_MAXW];    // [n_max][hq][d] on each instance
    uint32_t* qflag[PL_MAXW];         // [n_max]
    float* res_o[PL_MAXW];            // [m_max][W][hq][d]
    float* res_lse[PL_MAXW];          // [m_max][W][hq]
    uint32_t* res_flag[PL_MAXW];      // [m_max][W]
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_flag(const uint32_t* p, uint32_t want) {
    while (ld_acquire_sys(p) != want) {
        __nanosleep(64);
    }
}

}  // namespace dcp
