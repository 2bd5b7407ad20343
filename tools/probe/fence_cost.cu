// Probe: what a system-scope release costs inside a kernel (the MoE / exchange epilogues).
// Each kernel: 148 x 256 threads, every thread stores 64 B, then one release op per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fence_cost fence_cost.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(uint4* buf, unsigned* ctr) {
    uint4 v = make_uint4(threadIdx.x, blockIdx.x, 1, 2);
    uint4* p = buf + (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    p[0] = v; p[1] = v; p[2] = v; p[3] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        if (MODE == 1) asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        if (MODE == 2) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        if (MODE == 3) { __threadfence_system(); atomicAdd(ctr, 1); }
        if (MODE == 4) asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        if (MODE == 5) asm volatile("st.release.sys.global.u32 [%0], 1;" ::"l"(ctr) : "memory");
    }
}

template <int MODE>
float run(uint4* buf, unsigned* ctr, int reps, bool single) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 10; ++i) k<MODE><<<148, 256>>>(buf, ctr);
    cudaDeviceSynchronize();
    float best = 1e9, tot = 0;
    if (single) {
        for (int i = 0; i < reps; ++i) {
            cudaEventRecord(a);
            k<MODE><<<148, 256>>>(buf, ctr);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            tot += ms;
            if (ms < best) best = ms;
        }
        return tot / reps * 1e3f;
    }
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) k<MODE><<<148, 256>>>(buf, ctr);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps * 1e3f;
}

int main() {
    uint4* buf;
    unsigned* ctr;
    cudaMalloc(&buf, 148 * 256 * 64);
    cudaMalloc(&ctr, 4);
    const char* names[] = {"none", "red.release.sys", "red.release.gpu", "threadfence_system+atomic", "red.relaxed.sys",
                           "st.release.sys"};
    // clocks up: ~0.5 s of back-to-back launches before anything is timed
    for (int i = 0; i < 50000; ++i) k<0><<<148, 256>>>(buf, ctr);
    cudaDeviceSynchronize();
    float s[6], b[6];
    for (int pass = 0; pass < 2; ++pass) {
    s[0] = run<0>(buf, ctr, 200, true); b[0] = run<0>(buf, ctr, 2000, false);
    s[1] = run<1>(buf, ctr, 200, true); b[1] = run<1>(buf, ctr, 2000, false);
    s[2] = run<2>(buf, ctr, 200, true); b[2] = run<2>(buf, ctr, 2000, false);
    s[3] = run<3>(buf, ctr, 200, true); b[3] = run<3>(buf, ctr, 2000, false);
    s[4] = run<4>(buf, ctr, 200, true); b[4] = run<4>(buf, ctr, 2000, false);
    s[5] = run<5>(buf, ctr, 200, true); b[5] = run<5>(buf, ctr, 2000, false);
    }
    for (int i = 0; i < 6; ++i) printf("%-28s single-launch+events %.2f us   back-to-back %.2f us/launch\n", names[i], s[i], b[i]);
    return 0;
}
