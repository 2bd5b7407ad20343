// SPDX-License-Identifier: Apache-2.0
// Host-side definition of dcp_xchg shared by capi_xchg.cu, capi_attn.cu and capi_mla.cu.
#pragma once
#include "capi_common.cuh"
#include "exchange.cuh"

struct dcp_xchg {
    dcp_ctx* ctx = nullptr;
    dcp_xchg_config cfg{};      // normalised (q_dim, o_dim, q_elem_bytes, timeout_ms filled in)
    char* pool = nullptr;        // peer-visible pools (one cudaMalloc)
    size_t pool_bytes = 0;
    char* local = nullptr;       // local-only buffers
    dcp::XchgPeers host{};       // staged peer table
    dcp::XchgPeers* dev = nullptr;
    void* opened[dcp::PL_MAXW] = {};
    void* q_local = nullptr;
    float* out = nullptr;
    float* out_lse = nullptr;
    uint32_t* epoch = nullptr;
    uint32_t* err = nullptr;
    int32_t* exit_ticket = nullptr;  // fused step (dcp_decode_step_fused): grid exit counter
    bool committed = false;
};

namespace dcp {
// K2 / K3 with an explicit grid (an M-bucket's; the kernels stride over the device M count,
// so any grid is correct).  Stream-ordered, capturable.
int xchg_route_q_grid(dcp_xchg* x, const dcp_instance_view* v, int grid, cudaStream_t s);
int xchg_merge_grid(dcp_xchg* x, const dcp_instance_view* v, int grid, cudaStream_t s);
}  // namespace dcp
