// Probe (test tooling, not product): TMEM layout of the A operand of
// tcgen05.mma.cta_group::2.kind::f16 with A in TMEM (TS form), M = 128 (pair).
// B (K-major SW128, per CTA 16 rows) is the 16x16 identity, so D[m][n] = A[m][n % 16].
// A's TMEM words are filled with tags: run 0 tags both halves with the lane,
// run 1 tags lo = col, hi = 64 + col.  The host prints where A[m][k] was read from.
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>

#include "tc05.cuh"

using namespace dcp;

__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t col_elem) {
    const uint32_t byte = col_elem * 2;
    return row * 128 + ((((byte >> 4) ^ (row & 7)) & 7) << 4) + (byte & 15);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) ts_probe(float* out, int run) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const uint32_t base = smem_u32(sm);
    const uint32_t bar = base + 8192, tslot = base + 8192 + 64;
    const int cta = static_cast<int>(tc::cluster_ctarank());
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 16 * 64; i += 128) {
        const int r = i / 64, k = i % 64;
        *reinterpret_cast<__nv_bfloat16*>(sm + sw128(r, k)) = __float2bfloat16(k == r ? 1.f : 0.f);
    }
    tc::fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc<2>(tslot, 512);
    tc::fence_before_sync();
    tc::cluster_sync();
    tc::fence_after_sync();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sm + 8192 + 64);
    // A region: cols [256, 288)
    {
        uint32_t v[32];
        for (int c = 0; c < 32; ++c) {
            float lo, hi;
            if (run == 0) lo = hi = static_cast<float>(tid);
            else { lo = static_cast<float>(c); hi = static_cast<float>(64 + c); }
            __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
            v[c] = *reinterpret_cast<uint32_t*>(&h);
        }
        tc::tmem_st32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + 256, v);
        tc::tmem_wait_st();
    }
    tc::fence_before_sync();
    tc::cluster_sync();
    tc::fence_after_sync();
    if (cta == 0 && warp == 0) {
        const uint32_t id = tc::idesc_bf16_f32(128, 32, false, false);
        const uint64_t bd = tc::sdesc_sw128(base, 16, 1024);
        tc::mma2_bf16_ts_warp(tmem, tmem + 256, bd, id, 0);
        tc::commit2_mc_warp(bar, 0x3);
    }
    mbar_wait(bar, 0);
    tc::fence_after_sync();
    uint32_t v[32];
    tc::tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
    tc::tmem_wait_ld();
    for (int j = 0; j < 16; ++j) out[(cta * 128 + tid) * 16 + j] = __uint_as_float(v[j]);
    tc::fence_before_sync();
    tc::cluster_sync();
    if (warp == 0) tc::tmem_dealloc<2>(tmem, 512);
}

int main() {
    float* d;
    cudaMalloc(&d, 2 * 128 * 16 * 4);
    cudaFuncSetAttribute(ts_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    std::vector<float> o[2];
    for (int run = 0; run < 2; ++run) {
        cudaMemset(d, 0xff, 2 * 128 * 16 * 4);
        ts_probe<<<2, 128, 16384>>>(d, run);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        o[run].resize(2 * 128 * 16);
        cudaMemcpy(o[run].data(), d, o[run].size() * 4, cudaMemcpyDeviceToHost);
    }
    // D layout (pair M=128, N=32): CTA c, lane l<64 -> row 64c+l, n = col; lane 64+l -> row 64c+l, n = 16+col
    // D[m][n] = A[m][n % 16]
    for (int c = 0; c < 2; ++c)
        for (int l = 0; l < 128; l += 1) {
            if (!(l < 4 || (l >= 60 && l < 68) || l >= 124)) continue;
            printf("cta %d lane %3d (row %3d, n %s):", c, l, 64 * c + (l & 63), l < 64 ? "0-15" : "16-31");
            for (int j = 0; j < 16; ++j) printf(" %g/%g", o[0][(c * 128 + l) * 16 + j], o[1][(c * 128 + l) * 16 + j]);
            printf("\n");
        }
    return 0;
}
