// SPDX-License-Identifier: Apache-2.0
// Host-side definition of dcp_moe shared by capi_moe.cu and capi_graph.cu.
#pragma once
#include "capi_common.cuh"
#include "moe.cuh"

struct dcp_moe {
    dcp_ctx* ctx = nullptr;
    dcp_moe_config cfg{};
    char* pool = nullptr;
    char* local = nullptr;
    dcp::MoePeers host{};
    dcp::MoePeers* dev = nullptr;
    uint32_t* epoch = nullptr;
    uint32_t* err = nullptr;
    uint32_t host_epoch = 0;           // mirror of the device epoch (begin_step calls)
    const int32_t* m_count_dev = nullptr;
    bool received = false;
    bool committed = false;
    void* opened[dcp::PL_MAXW] = {};
};
