// SPDX-License-Identifier: Apache-2.0
// Host-side definition of dcp_xchg shared by capi_xchg.cu and capi_attn.cu.
#pragma once
#include "capi_common.cuh"
#include "exchange.cuh"

struct dcp_xchg {
    dcp_ctx* ctx = nullptr;
    dcp_xchg_config cfg{};
    char* pool = nullptr;        // peer-visible pools (one cudaMalloc)
    size_t pool_bytes = 0;
    char* local = nullptr;       // local-only buffers
    dcp::XchgPeers host{};       // staged peer table
    dcp::XchgPeers* dev = nullptr;
    void* opened[dcp::PL_MAXW] = {};
    // offsets within a pool (identical on every instance)
    size_t off_qrecv = 0, off_qflag = 0, off_res_o = 0, off_res_lse = 0, off_res_flag = 0;
    void* q_local = nullptr;
    float* out = nullptr;
    float* out_lse = nullptr;
    uint32_t* epoch = nullptr;
};
