// SPDX-License-Identifier: Apache-2.0
// Host-side definition of dcp_planner shared by capi_planner.cu and capi_dropin.cu.
#pragma once
#include <cuda_bf16.h>

#include <unordered_map>
#include <vector>

#include "capi_common.cuh"
#include "planner.cuh"
#include "routing.cuh"

struct dcp_planner {
    dcp_ctx* ctx = nullptr;
    dcp_planner_config cfg{};
    dcp::PlannerState st{};
    dcp::RoutingOut ro{};
    std::vector<void*> owned;
    int32_t* arena2_inst = nullptr;
    int32_t* arena2_frame = nullptr;
    uint8_t* arena2_fill = nullptr;
    int64_t* d_new_off = nullptr;
    int32_t* d_io_slots = nullptr;   // staging
    int64_t* d_io_ids = nullptr;
    int64_t* d_io_lens = nullptr;
    int32_t* d_io_out = nullptr;
    std::unordered_map<int64_t, int32_t> slot_of;
    std::vector<int32_t> free_slots;
    std::vector<int64_t> id_of_slot;
    int64_t arena_top_host = 0;      // upper bound between syncs
    int64_t waiting_pages_bound = 0; // sum over queued requests of their max arena demand
    std::vector<int64_t> queued_len; // per slot (for the bound)
    std::vector<uint8_t> is_active;  // host mirror of state == ACTIVE (set by step results / allocate)
    int32_t queued = 0;
    struct Retired {
        int32_t k, moe;
        int32_t kv[dcp::PL_MAXK];
        int64_t split[dcp::PL_MAXK];
    };
    // Finished requests keep their Placement (Request::placement is not cleared
    // by pt_free, page_table.cpp:51-66), so placement queries still answer.
    std::unordered_map<int64_t, Retired> retired;
    cudaStream_t stream = nullptr;
    int last_launches = 0;
    bool routing_valid = false;
    uint64_t generation = 0;         // bumped when device pointers inside `st` change (arena compaction)
    __nv_bfloat16** d_pools = nullptr;  // K8 pool table
};

namespace dcp {
int planner_sync_arena_top(dcp_planner* pl);
int planner_compact(dcp_planner* pl);
}  // namespace dcp
