// SPDX-License-Identifier: Apache-2.0
// Shared C-ABI plumbing: error state, context object, CUDA error mapping.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "dcp_capi.h"

namespace dcp {

void set_error(const char* fmt, ...);

#define DCP_CUDA_TRY(expr)                                                              \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            ::dcp::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(e_)); \
            return DCP_E_CUDA;                                                          \
        }                                                                               \
    } while (0)

#define DCP_REQUIRE(cond, code, ...)        \
    do {                                    \
        if (!(cond)) {                      \
            ::dcp::set_error(__VA_ARGS__);  \
            return (code);                  \
        }                                   \
    } while (0)

struct TmapCacheEntry {
    const void* base = nullptr;
    int64_t frames = 0;
    int hkv = 0;
    int d = 0;
    bool split = false;
    int page = 16;
    CUtensorMap map;
};

// Launch with programmatic stream serialization (PDL): the kernel may start while its stream
// predecessor is still running and must pdl_wait() (ptx.cuh) before reading that kernel's
// output; the launch gap between dependent short kernels disappears.  Graph-capturable.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace dcp

// Sets K1's dynamic shared-memory attribute for (hkv, group) outside any capture.
int dcp_attn_prepare(struct dcp_ctx* ctx, int hkv, int group, int page);

struct dcp_ctx {
    int device = 0;
    int num_sms = 0;
    int cc_major = 0, cc_minor = 0;
    dcp::TmapCacheEntry kv_maps[4];
    int kv_map_next = 0;
};

// NVTX range over one C-ABI call (SURVEY §5 tracing): a profiler (nsys / ncu --nvtx) sees each
// host-side phase of the step (planner, routing, attention, exchange, MoE) as a named range.
// NVTX v3 is header-only; without an attached tool a push / pop is one predictable branch.
struct DcpNvtxRange {
    explicit DcpNvtxRange(const char* name) { nvtxRangePushA(name); }
    ~DcpNvtxRange() { nvtxRangePop(); }
    DcpNvtxRange(const DcpNvtxRange&) = delete;
    DcpNvtxRange& operator=(const DcpNvtxRange&) = delete;
};
#define DCP_NVTX(name) DcpNvtxRange dcp_nvtx_range_(name)
