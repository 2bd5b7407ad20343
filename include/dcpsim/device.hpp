// SPDX-License-Identifier: Apache-2.0
//
// dcpsim drop-in: device binding.  Not part of the reference API; this is the
// seam between the reference-shaped C++ surface and the sm_100a C ABI
// (include/dcp_capi.h).  All planning, allocation, routing and attention work
// behind the dcpsim functions runs on the device selected here.
#pragma once

#include <memory>

#include "dcp_capi.h"

#pragma GCC visibility push(default)

namespace dcpsim::device {

// Process-wide context on CUDA device DCP_DEVICE (default 0), created lazily.
dcp_ctx* context();
// Select the device before first use (throws ConfigError afterwards).
void set_device(int device);
// Map a DCP_E_* status to the matching dcpsim exception (no-op for 0).
void check(int rc);

// RAII owner of a device planner bound to one ClusterState.
struct Planner {
    dcp_planner* handle = nullptr;
    int world = 0;
    long long page_size = 0;
    long long capacity = 0;
    ~Planner();
};

}  // namespace dcpsim::device

#pragma GCC visibility pop
