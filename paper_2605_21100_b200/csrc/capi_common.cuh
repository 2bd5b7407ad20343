// SPDX-License-Identifier: Apache-2.0
// Shared C-ABI plumbing: error state, context object, CUDA error mapping.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

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
