// Probe (test tooling, not product): issue rate and throughput of 2-CTA
// (measured: an accumulating M=128-pair MMA costs ~120 ns whatever N <= 256 and
// however many accumulators are interleaved; accumulate=0 MMAs overlap)
//
// tcgen05.mma (kind::f16, SS) at the MLA kernel's shapes, with a commit every
// `per_commit` MMAs.  One cluster of 2 per TPC, all SMs busy.
#include <cuda_bf16.h>
#include <cstdio>

#include "tc05.cuh"

using namespace dcp;

__device__ __forceinline__ long long gt() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_rate(long long* out, int n_mma, int per_commit, int N, int b_mn, int nd, int nw) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const uint32_t base = smem_u32(sm);
    const uint32_t bar0 = base + 65536, tslot = bar0 + 64;
    const int cta = static_cast<int>(tc::cluster_ctarank());
    const int warp = threadIdx.x >> 5;
    const uint32_t bar = bar0 + 8 * (warp > 0 ? warp - 1 : 0);
    for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    tc::fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (int k = 0; k < 4; ++k) mbar_init(bar0 + 8 * k, 1);
        fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc<2>(tslot, 512);
    tc::fence_before_sync();
    tc::cluster_sync();
    tc::fence_after_sync();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sm + 65536 + 64);
    if (cta == 0 && warp >= 1 && warp <= nw) {
        const uint32_t id = tc::idesc_bf16_f32(128, N, false, b_mn != 0);
        const uint64_t ad = tc::sdesc_sw128(base, 16, 1024);
        const uint64_t bd = tc::sdesc_sw128(base + 32768, b_mn ? 4096 : 16, 1024);
        const long long t0 = gt();
        int commits = 0;
        for (int i = 0; i < n_mma; ++i) {
            tc::mma2_bf16_ss_warp(tmem + ((warp - 1) * nd + i % nd) * (N / 2), ad + 2 * (i & 3), bd + 2 * (i & 3), id, i >= nd);
            if ((i + 1) % per_commit == 0) {
                tc::commit2_mc_warp(bar, 0x3);
                ++commits;
            }
        }
        const long long t1 = gt();
        tc::commit2_mc_warp(bar, 0x3);
        ++commits;
        // wait for the last commit's phase
        if ((threadIdx.x & 31) == 0) {
            // phases completed so far = commits; the last one completes phase (commits-1)
            mbar_wait(bar, (commits - 1) & 1);
        }
        __syncwarp();
        const long long t2 = gt();
        if ((threadIdx.x & 31) == 0 && blockIdx.x == 0 && warp == 1) {
            out[0] = t1 - t0;
            out[1] = t2 - t0;
        }
    }
    tc::fence_before_sync();
    tc::cluster_sync();
    if (warp == 0) tc::tmem_dealloc<2>(tmem, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 65536 + 2048;
    cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    struct C { int n, pc, N, mn, nd, nw; } cfgs[] = {{3600, 36, 128, 0, 1, 1}, {3600, 36, 128, 0, 1, 2}, {3600, 36, 128, 0, 1, 3},
                                             {1600, 16, 256, 1, 1, 1}, {1600, 16, 256, 1, 1, 2}, {3600, 36, 64, 0, 1, 1}, {3600, 36, 64, 0, 1, 3}};
    for (auto c : cfgs) {
        mma_rate<<<sms & ~1, 128, smem>>>(d, c.n, c.pc, c.N, c.mn, c.nd, c.nw);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        const double macs = double(c.n) * c.nw * 128 * c.N * 16;  // per pair
        printf("warps=%d nd=%d N=%d %s, %d MMAs, commit every %4d: issue %7.1f ns/MMA, complete %7.1f ns/MMA, %6.1f TFLOP/s chip %s\n",
               c.nw, c.nd, c.N, c.mn ? "B MN-major" : "B K-major", c.n, c.pc, double(h[0]) / c.n, double(h[1]) / c.n,
               2 * macs * (sms / 2) / (h[1] * 1e-9) / 1e12, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
