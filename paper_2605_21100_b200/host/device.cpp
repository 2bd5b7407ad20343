// SPDX-License-Identifier: Apache-2.0
// dcpsim drop-in: process-wide device context and status -> exception mapping.
#include <cstdlib>
#include <mutex>
#include <string>

#include "dcpsim/device.hpp"
#include "dcpsim/types.hpp"

namespace dcpsim::device {

namespace {
std::mutex g_mu;
dcp_ctx* g_ctx = nullptr;
int g_device = -1;
}  // namespace

void check(int rc) {
    if (rc == DCP_OK) return;
    const std::string msg = std::string("dcp: ") + dcp_last_error();
    switch (rc) {
        case DCP_E_INSUFFICIENT_FRAMES: throw InsufficientFrames(msg);
        case DCP_E_UNKNOWN_REQUEST: throw UnknownRequest(msg);
        case DCP_E_UNKNOWN_PAGE: throw UnknownPage(msg);
        case DCP_E_INCONSISTENT: throw InconsistentPlacement(msg);
        case DCP_E_SHAPE_OVERFLOW: throw ShapeOverflow(msg);
        case DCP_E_EMPTY_SHARD: throw EmptyShard(msg);
        case DCP_E_CONFIG: throw ConfigError(msg);
        default: throw SimError(msg + " (status " + std::to_string(rc) + ")");
    }
}

void set_device(int device) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_ctx && device != g_device) throw ConfigError("dcpsim device already initialised");
    g_device = device;
}

dcp_ctx* context() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_ctx) {
        int dev = g_device;
        if (dev < 0) {
            const char* e = std::getenv("DCP_DEVICE");
            dev = e ? std::atoi(e) : 0;
        }
        dcp_ctx* c = nullptr;
        check(dcp_ctx_create(dev, &c));
        g_ctx = c;
        g_device = dev;
    }
    return g_ctx;
}

Planner::~Planner() {
    if (handle) dcp_planner_destroy(handle);
}

}  // namespace dcpsim::device
