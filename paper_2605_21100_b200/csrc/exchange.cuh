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
// Step protocol (every instance calls begin_step once per step):
//   * Flags carry the step's epoch e, so graph replay needs no flag reset.
//   * Every receive buffer and flag exists twice, selected by e & 1: a peer
//     still reading step e-1's slots is never overwritten by step e.
//   * begin_step(e) first publishes "done = e-1" in this instance's pool (all of
//     its step e-1 kernels finished: stream order), then waits until every peer
//     published done >= e-2.  So no instance runs more than one step ahead of
//     any peer, and step e's writes into parity e & 1 can only meet readers of
//     step e (step e-2, the previous user of that parity, is over everywhere).
//   * Every flag wait is bounded (timeout_ns, globaltimer).  A wait that times
//     out records {code, where, want, seen} in the instance's error word, and
//     every later wait of that instance bails out at once; the kernels still run
//     to completion (their outputs are garbage) and the host reads the error
//     with dcp_xchg_status / dcp_moe_status.  A lost or mis-epoched flag is an
//     error code, never a hung GPU.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>

#include "limits.cuh"

namespace dcp {

// error word layout (4 x u32): code, where, want, seen
enum : uint32_t { XERR_NONE = 0, XERR_TIMEOUT = 1 };
// `where` = site << 24 | peer << 16 | (row & 0xffff)
enum : uint32_t {
    SITE_FENCE = 1, SITE_K1_Q = 2, SITE_K3_RES = 3, SITE_MOE_RX = 4, SITE_MOE_CB = 5, SITE_K10_Q = 6
};

struct WaitCtl {
    uint32_t* err;        // local [4]
    uint64_t timeout_ns;
};

struct XchgPeers {
    int32_t W, self, hq, q_dim, o_dim, q_bytes, n_max, m_max;
    uint32_t* epoch;      // local, bumped per step
    WaitCtl wc;
    char* base[PL_MAXW];  // each instance's pool, as addressable from this device
    // pool layout (identical on every instance): per parity p in {0, 1}
    //   qrecv   [n_max][hq][q_dim] x q_bytes   at off_qrecv   + p * sz_qrecv
    //   qflag   [n_max] u32                    at off_qflag   + p * sz_qflag
    //   res_o   [m_max][W][hq][o_dim] fp32     at off_res_o   + p * sz_res_o
    //   res_lse [m_max][W][hq] fp32            at off_res_lse + p * sz_res_lse
    //   res_flag[m_max][W] u32                 at off_res_flag+ p * sz_res_flag
    //   done    u32 (last completed epoch)     at off_done
    uint64_t off_qrecv, off_qflag, off_res_o, off_res_lse, off_res_flag, off_done;
    uint64_t sz_qrecv, sz_qflag, sz_res_o, sz_res_lse, sz_res_flag;
};

__device__ __forceinline__ char* xq_recv(const XchgPeers& x, int s, uint32_t ep) {
    return x.base[s] + x.off_qrecv + (ep & 1) * x.sz_qrecv;
}
__device__ __forceinline__ uint32_t* xq_flag(const XchgPeers& x, int s, uint32_t ep) {
    return reinterpret_cast<uint32_t*>(x.base[s] + x.off_qflag + (ep & 1) * x.sz_qflag);
}
__device__ __forceinline__ float* xres_o(const XchgPeers& x, int s, uint32_t ep) {
    return reinterpret_cast<float*>(x.base[s] + x.off_res_o + (ep & 1) * x.sz_res_o);
}
__device__ __forceinline__ float* xres_lse(const XchgPeers& x, int s, uint32_t ep) {
    return reinterpret_cast<float*>(x.base[s] + x.off_res_lse + (ep & 1) * x.sz_res_lse);
}
__device__ __forceinline__ uint32_t* xres_flag(const XchgPeers& x, int s, uint32_t ep) {
    return reinterpret_cast<uint32_t*>(x.base[s] + x.off_res_flag + (ep & 1) * x.sz_res_flag);
}
__device__ __forceinline__ uint32_t* xdone(const XchgPeers& x, int s) {
    return reinterpret_cast<uint32_t*>(x.base[s] + x.off_done);
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Spin until poll(&seen) returns true, at most wc.timeout_ns.  Returns false on timeout or
// when an earlier wait of this instance already failed (the error word is set): callers carry
// on with whatever data is there, so every kernel still terminates.
template <class Poll>
__device__ __forceinline__ bool wait_until(Poll poll, uint32_t want, const WaitCtl& wc, uint32_t where) {
    uint32_t seen = 0;
    if (poll(seen)) return true;
    const uint64_t t0 = globaltimer_ns();
    for (;;) {
        __nanosleep(64);
        if (poll(seen)) return true;
        if (*reinterpret_cast<volatile uint32_t*>(wc.err) != XERR_NONE) return false;
        if (globaltimer_ns() - t0 > wc.timeout_ns) {
            if (atomicCAS(wc.err, XERR_NONE, XERR_TIMEOUT) == XERR_NONE) {
                wc.err[1] = where;
                wc.err[2] = want;
                wc.err[3] = seen;
                __threadfence_system();
            }
            return false;
        }
    }
}

// *p == want, or *p >= want in serial-number order when `at_least`.
__device__ __forceinline__ bool wait_flag(const uint32_t* p, uint32_t want, const WaitCtl& wc, uint32_t where,
                                          bool at_least = false) {
    return wait_until(
        [&](uint32_t& seen) {
            seen = ld_acquire_sys(p);
            return at_least ? static_cast<int32_t>(seen - want) >= 0 : seen == want;
        },
        want, wc, where);
}

// begin_step: publish done = e-1 in our own pool, wait for every peer's done >= e-2, then
// advance the epoch.  One warp; lane s watches peer s.  done_of(s) -> u32* of s's done word.
// The done store needs no release fence (a MEMBAR.SYS costs microseconds): every access of
// step e-1 belongs to kernels that completed before this one started (stream order), so
// nothing of ours can be reordered after it.  The peers' done words are read with acquire
// loads, which order this instance's later stores into their pools.
template <class DoneOf>
__device__ __forceinline__ void step_fence(uint32_t* epoch, DoneOf done_of, int W, int self, const WaitCtl& wc) {
    const uint32_t e = *epoch + 1;
    const int lane = threadIdx.x & 31;
    if (lane == 0) st_relaxed_sys(done_of(self), e - 1);
    __syncwarp();
    for (int s = lane; s < W; s += 32)
        if (s != self) wait_flag(done_of(s), e - 2, wc, (SITE_FENCE << 24) | (s << 16), true);
    __syncwarp();
    if (lane == 0) *epoch = e;
}

}  // namespace dcp
