// Probe (test tooling, not product): pins the tcgen05 facts the MLA kernel
// relies on, on the real B200.
//   T1  cta_group::1  M=128 N=64  K=64, A,B K-major SW128     (S = Q K^T form)
//   T2  cta_group::2  M=128 N=128 K=64, A,B K-major SW128     (pair QK^T)
//   T3  cta_group::2  M=128 N=256 K=32, A K-major, B MN-major (pair P V)
// For T2/T3 it tests the hypothesised TMEM layout of the pair accumulator:
//   CTA c, lane l < 64, col j  -> D[64c + l][j]
//   CTA c, lane 64 + l, col j  -> D[64c + l][N/2 + j]
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++20 -I paper_2605_21100_b200/csrc tools/probe/tc05_probe.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc05.cuh"

using namespace dcp;

__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t col_elem) {
    // byte offset of bf16 element (row, col) in a 128-B-row, 128B-swizzled tile
    const uint32_t byte = col_elem * 2;
    return row * 128 + ((((byte >> 4) ^ (row & 7)) & 7) << 4) + (byte & 15);
}

struct Args {
    const __nv_bfloat16* A;  // [M][K] row-major (pair-total rows)
    const __nv_bfloat16* B;  // T1/T2: [N][K] row-major; T3: [K][N] row-major (tokens x dims)
    float* out;              // [ncta][128][ncols]
    int test, M, N, K, ncols;
};

template <int NCTA>
__global__ void __launch_bounds__(128, 1) probe_kernel(Args a) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const uint32_t base = smem_u32(sm);
    const uint32_t a_off = 0, b_off = 32768;
    const uint32_t bar = base + 65536, tslot = base + 65536 + 64;
    const int cta = NCTA == 2 ? static_cast<int>(tc::cluster_ctarank()) : 0;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int rows_a = a.M / NCTA;

    // A: rows [cta*rows_a, +rows_a), K-major, one 64-wide K box (K <= 64)
    for (int i = tid; i < rows_a * 64; i += 128) {
        const int r = i / 64, k = i % 64;
        __nv_bfloat16 v = k < a.K ? a.A[(cta * rows_a + r) * a.K + k] : __float2bfloat16(0.f);
        *reinterpret_cast<__nv_bfloat16*>(sm + a_off + sw128(r, k)) = v;
    }
    if (a.test != 3) {  // B K-major: rows (N) [cta*N/NCTA, ...)
        const int rows_b = a.N / NCTA;
        for (int i = tid; i < rows_b * 64; i += 128) {
            const int r = i / 64, k = i % 64;
            __nv_bfloat16 v = k < a.K ? a.B[(cta * rows_b + r) * a.K + k] : __float2bfloat16(0.f);
            *reinterpret_cast<__nv_bfloat16*>(sm + b_off + sw128(r, k)) = v;
        }
    } else {  // B MN-major: this CTA's N/2 dims as boxes of [K tokens][64 dims]
        const int nb = a.N / NCTA / 64;
        for (int i = tid; i < nb * a.K * 64; i += 128) {
            const int bx = i / (a.K * 64), rem = i % (a.K * 64), t = rem / 64, d = rem % 64;
            const int n = cta * (a.N / NCTA) + bx * 64 + d;
            *reinterpret_cast<__nv_bfloat16*>(sm + b_off + bx * (a.K * 128) + sw128(t, d)) = a.B[t * a.N + n];
        }
    }
    tc::fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc<NCTA>(tslot, 512);
    tc::fence_before_sync();
    if (NCTA == 2) tc::cluster_sync(); else __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sm + 65536 + 64);

    if (cta == 0 && tid == 0) {
        if (a.test != 3) {
            const uint32_t id = tc::idesc_bf16_f32(a.M, a.N, false, false);
            for (int k = 0; k < a.K / 16; ++k) {
                const uint64_t ad = tc::sdesc_sw128(base + a_off + 32 * k, 16, 1024);
                const uint64_t bd = tc::sdesc_sw128(base + b_off + 32 * k, 16, 1024);
                tc::mma_bf16_ss<NCTA>(tmem, ad, bd, id, k > 0);
            }
        } else {
            const uint32_t id = tc::idesc_bf16_f32(a.M, a.N, false, true);
            for (int k = 0; k < a.K / 16; ++k) {
                const uint64_t ad = tc::sdesc_sw128(base + a_off + 32 * k, 16, 1024);
                const uint64_t bd = tc::sdesc_sw128(base + b_off + 16 * 128 * k, a.K * 128, 1024);
                tc::mma_bf16_ss<NCTA>(tmem, ad, bd, id, k > 0);
            }
        }
        if (NCTA == 2) tc::commit2_mc(bar, 0x3); else tc::commit1(bar);
    }
    tc::mbar_wait_cluster(bar, 0);
    tc::fence_after_sync();
    for (int c0 = 0; c0 < a.ncols; c0 += 32) {
        uint32_t v[32];
        tc::tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
        tc::tmem_wait_ld();
        const int lane_row = warp * 32 + (tid & 31);
        for (int j = 0; j < 32; ++j)
            a.out[(static_cast<size_t>(cta) * 128 + lane_row) * a.ncols + c0 + j] = __uint_as_float(v[j]);
    }
    tc::fence_before_sync();
    if (NCTA == 2) tc::cluster_sync(); else __syncthreads();
    if (warp == 0) tc::tmem_dealloc<NCTA>(tmem, 512);
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

static int run(int test) {
    const int ncta = test == 1 ? 1 : 2;
    int M = 128, N, K;
    if (test == 1) { N = 64; K = 64; }
    else if (test == 2) { N = 128; K = 64; }
    else { N = 256; K = 32; }
    const int ncols = test == 1 ? N : N / 2;
    std::vector<__nv_bfloat16> A(M * K), B(N * K);
    std::vector<float> Af(M * K), Bf(N * K);
    srand(1234 + test);
    for (int i = 0; i < M * K; ++i) { Af[i] = bf(static_cast<float>(rand() % 7 - 3)); A[i] = __float2bfloat16(Af[i]); }
    for (int i = 0; i < N * K; ++i) { Bf[i] = bf(static_cast<float>(rand() % 7 - 3)); B[i] = __float2bfloat16(Bf[i]); }
    // D[m][n]
    std::vector<double> D(M * N, 0.0);
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k)
                s += Af[m * K + k] * (test == 3 ? Bf[k * N + n] : Bf[n * K + k]);
            D[m * N + n] = s;
        }
    __nv_bfloat16 *dA, *dB;
    float* dO;
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dO, ncta * 128 * ncols * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(dO, 0xff, ncta * 128 * ncols * 4);
    Args a{dA, dB, dO, test, M, N, K, ncols};
    const int smem = 65536 + 1024 + 128;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncta);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ncta;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (ncta == 1) {
        cudaFuncSetAttribute(probe_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&cfg, probe_kernel<1>, a);
    } else {
        cudaFuncSetAttribute(probe_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&cfg, probe_kernel<2>, a);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("T%d: CUDA error %s\n", test, cudaGetErrorString(e)); return 1; }
    std::vector<float> O(ncta * 128 * ncols);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0, shown = 0;
    for (int c = 0; c < ncta; ++c)
        for (int l = 0; l < 128; ++l)
            for (int j = 0; j < ncols; ++j) {
                int m, n;
                if (ncta == 1) { m = l; n = j; }
                else { m = 64 * c + (l & 63); n = (l < 64 ? 0 : N / 2) + j; }
                const float got = O[(c * 128 + l) * ncols + j];
                if (got != static_cast<float>(D[m * N + n])) {
                    if (shown++ < 6) {
                        // find where the value would come from
                        int fm = -1, fn = -1;
                        for (int mm = 0; mm < M && fm < 0; ++mm)
                            for (int nn = 0; nn < N; ++nn)
                                if (static_cast<float>(D[mm * N + nn]) == got) { fm = mm; fn = nn; break; }
                        printf("  T%d cta %d lane %d col %d: got %g want D[%d][%d]=%g (first match D[%d][%d])\n", test, c, l,
                               j, got, m, n, D[m * N + n], fm, fn);
                    }
                    ++bad;
                }
            }
    printf("T%d: %s (%d mismatches of %d)\n", test, bad ? "FAIL" : "PASS", bad, ncta * 128 * ncols);
    cudaFree(dA); cudaFree(dB); cudaFree(dO);
    return bad != 0;
}

int main() {
    int rc = 0;
    for (int t = 1; t <= 3; ++t) rc |= run(t);
    return rc;
}
