// Probe (test tooling, not product): HBM streaming bandwidth of TMA loads as a
// function of box size and bytes in flight per SM, random 16-token frames like the
// paged caches.  One CTA per SM; warp 0 lane 0 issues 2-D TMA boxes of R rows x 128 B
// into a ring of NS stages of STAGE bytes; warp 1 lane 0 consumes (waits full,
// releases empty).  Prints GB/s per configuration.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++20 -I paper_2605_21100_b200/csrc tools/probe/tma_bw.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace dcp;

struct P {
    int rows_per_box;   // box rows (each 128 B)
    int boxes_per_stage;
    int ns;             // stages
    int iters;          // stages per CTA
    int nframes;        // frames of 16 rows in the buffer
    int issuers;        // producer threads (lanes of warp 0) issuing boxes of one stage in parallel
};

__global__ void __launch_bounds__(64, 1) tma_bw_kernel(const __grid_constant__ CUtensorMap map, P p) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const uint32_t base = smem_u32(sm);
    const int stage_bytes = p.rows_per_box * 128 * p.boxes_per_stage;
    const uint32_t bars = base + p.ns * stage_bytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.ns; ++s) {
            mbar_init(bars + 8 * s, 1);
            mbar_init(bars + 8 * (p.ns + s), 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t rng = 12345u + blockIdx.x * 7919u;
    if (warp == 0 && lane < p.issuers) {
        for (int it = 0; it < p.iters; ++it) {
            const int s = it % p.ns;
            if (lane == 0) {
                mbar_wait(bars + 8 * (p.ns + s), ((it / p.ns) & 1) ^ 1);
                mbar_arrive_expect_tx(bars + 8 * s, stage_bytes);
            }
            __syncwarp((1u << p.issuers) - 1);
            for (int b = lane; b < p.boxes_per_stage; b += p.issuers) {
                rng = rng * 1664525u + 1013904223u;
                const int frame = (rng >> 8) % p.nframes;
                tma_load_2d(base + s * stage_bytes + b * p.rows_per_box * 128, &map, 0, frame * 16, bars + 8 * s,
                            l2_policy_evict_first());
            }
        }
    } else if (warp == 1 && lane == 0) {
        for (int it = 0; it < p.iters; ++it) {
            const int s = it % p.ns;
            mbar_wait(bars + 8 * s, (it / p.ns) & 1);
            mbar_arrive(bars + 8 * (p.ns + s));
        }
    }
}

int main() {
    const size_t bytes = size_t(4) << 30;  // 4 GB buffer of 16-row frames (128 B rows)
    void* buf;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("malloc failed\n"); return 1; }
    cudaMemset(buf, 0, bytes);
    const int nframes = static_cast<int>(bytes / (16 * 128));
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(tma_bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    struct C { int rows, bps, ns, issuers; };
    std::vector<C> cfgs = {
        {16, 4, 15, 1}, {16, 4, 24, 1}, {16, 8, 12, 1}, {16, 8, 12, 4}, {16, 4, 15, 4},
        {64, 1, 15, 1}, {64, 1, 24, 1}, {64, 2, 12, 1}, {128, 1, 12, 1}, {256, 1, 6, 1}, {256, 2, 3, 1},
        {16, 16, 6, 1}, {16, 16, 6, 8}, {32, 8, 6, 1},
    };
    for (auto c : cfgs) {
        CUtensorMap map;
        cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(nframes) * 16};
        cuuint64_t strides[1] = {128};
        cuuint32_t box[2] = {64, static_cast<cuuint32_t>(c.rows)};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); continue; }
        const int stage = c.rows * 128 * c.bps;
        P p{c.rows, c.bps, c.ns, 0, nframes, c.issuers};
        p.iters = static_cast<int>((size_t(3) << 30) / sms / stage);  // ~3 GB total
        const int smem = c.ns * stage + 16 * c.ns + 2048;
        if (smem > 227 * 1024) { printf("skip (smem)\n"); continue; }
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        tma_bw_kernel<<<sms, 64, smem>>>(map, p);
        cudaEventRecord(e0);
        tma_bw_kernel<<<sms, 64, smem>>>(map, p);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double tot = double(p.iters) * stage * sms;
        printf("box %3d rows (%5d B) x %2d per stage, %2d stages (%6d B in flight), %d issuer(s): %7.1f GB/s %s\n",
               c.rows, c.rows * 128, c.bps, c.ns, c.ns * stage, c.issuers, tot / ms / 1e6,
               err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
    return 0;
}
