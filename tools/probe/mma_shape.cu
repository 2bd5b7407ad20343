// Probe (test tooling, not product): time per DEPENDENT tcgen05.mma (one
// accumulator, one issuing warp, SS mode, bf16 -> f32) as a function of the
// MMA shape and cta_group, to choose K10's decomposition.
//   cg1: M in {64, 128}, N in {64, 128, 256}
//   cg2: M in {128, 256} (pair-total), N in {64, 128, 256}
// Also: 2 and 4 independent accumulator chains issued by one warp (interleaved).
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++20 -I paper_2605_21100_b200/csrc tools/probe/mma_shape.cu -o tools/probe/_bin/mma_shape
#include <cuda_bf16.h>
#include <cstdio>

#include "tc05.cuh"

using namespace dcp;

__device__ __forceinline__ long long gt() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void mma1_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit1_warp(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
        : "memory");
}

template <int CG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    mma_shape(long long* out, int n_mma, int M, int N, int nchains, int nw) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const uint32_t base = smem_u32(sm);
    const uint32_t bar = base + 131072, tslot = bar + 64;
    const int cta = static_cast<int>(tc::cluster_ctarank());
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    tc::fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (int k = 0; k < 4; ++k) mbar_init(bar + 8 * k, 1);
        fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc<CG>(tslot, 512);
    tc::fence_before_sync();
    tc::cluster_sync();
    tc::fence_after_sync();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sm + 131072 + 64);
    const bool issuer = (CG == 1) ? (warp >= 1 && warp <= nw) : (cta == 0 && warp >= 1 && warp <= nw);
    if (issuer) {
        const uint32_t id = tc::idesc_bf16_f32(M, N, false, false);
        const uint64_t ad = tc::sdesc_sw128(base, 16, 1024);
        const uint64_t bd = tc::sdesc_sw128(base + 65536, 16, 1024);
        // accumulator columns per chain: N (cg1 M=128 / cg2 M=256), N/2 folded (cg2 M=128), N (cg1 M=64)
        const int cols = (CG == 2 && M == 128) ? N / 2 : N;
        const long long t0 = gt();
        for (int i = 0; i < n_mma; ++i) {
            const int ch = (warp - 1) * nchains + i % nchains;
            const uint32_t d = tmem + ch * cols;
            if constexpr (CG == 1)
                mma1_warp(d, ad + 2 * (i & 3), bd + 2 * (i & 3), id, i >= nchains);
            else
                tc::mma2_bf16_ss_warp(d, ad + 2 * (i & 3), bd + 2 * (i & 3), id, i >= nchains);
        }
        const long long t1 = gt();
        if constexpr (CG == 1)
            commit1_warp(bar + 8 * (warp - 1));
        else
            tc::commit2_mc_warp(bar + 8 * (warp - 1), 0x1);
        if ((threadIdx.x & 31) == 0) mbar_wait(bar + 8 * (warp - 1), 0);
        __syncwarp();
        const long long t2 = gt();
        if ((threadIdx.x & 31) == 0 && blockIdx.x == 0 && warp == 1) {
            out[0] = t1 - t0;
            out[1] = t2 - t0;
        }
    }
    tc::fence_before_sync();
    tc::cluster_sync();
    if (warp == 0) tc::tmem_dealloc<CG>(tmem, 512);
}

template <int CG>
void run(long long* d, int sms, int M, int N, int nch, int nw = 1) {
    const int cols = (CG == 2 && M == 128) ? N / 2 : N;
    if (cols * nch * nw > 512) return;
    const int smem = 131072 + 2048;
    cudaFuncSetAttribute(mma_shape<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int n = 2400;
    mma_shape<CG><<<sms & ~1, 192, smem>>>(d, n, M, N, nch, nw);  // warm
    cudaDeviceSynchronize();
    mma_shape<CG><<<sms & ~1, 192, smem>>>(d, n, M, N, nch, nw);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    // MACs per MMA instruction: M x N x 16 (M pair-total for cg2)
    const double units = (CG == 1) ? sms : sms / 2;  // issuing units chip-wide
    const double flops = 2.0 * M * N * 16 * n * units * nw;
    printf("cg%d M=%3d N=%3d chains=%d warps=%d: issue %6.1f ns/MMA, complete %6.1f ns/MMA (%5.0f cyc @1.9GHz), chip %7.1f TFLOP/s %s\n",
           CG, M, N, nch, nw, double(h[0]) / n, double(h[1]) / n, double(h[1]) / n * 1.9, flops / (h[1] * 1e-9) / 1e12,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int nw : {2, 3, 4}) {
        for (int N : {64, 128, 256}) {
            run<1>(d, sms, 128, N, 1, nw);
            run<2>(d, sms, 128, N, 1, nw);
            run<2>(d, sms, 256, N, 1, nw);
        }
    }
    for (int nch : {1}) {
        for (int N : {64, 128, 256}) {
            run<1>(d, sms, 64, N, nch);
            run<1>(d, sms, 128, N, nch);
            run<2>(d, sms, 128, N, nch);
            run<2>(d, sms, 256, N, nch);
        }
    }
    return 0;
}
