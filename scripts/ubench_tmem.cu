// Microbenchmark: TMEM -> register load throughput (tcgen05.ld.32x32b.x32), W warps per CTA
// (warp w reads lane quadrant w % 4), one CTA per SM.  Usage: ubench_tmem <warps> <x64 0/1>
#include "../paper_2603_29494_b200/csrc/common.cuh"
#include <cstdio>
#include <cstdlib>

using namespace va;
constexpr int REPS = 4096;

__global__ void __launch_bounds__(512, 1) kern(int two, unsigned long long* out, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot + (((warp & 3) * 32u) << 16) + 64u * (warp >> 2);
    float acc = 0.f;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int r = 0; r < REPS; ++r) {
        uint32_t a[32], b[32];
        tmem_ld32(tm, a);
        if (two) tmem_ld32(tm + 32, b);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += __uint_as_float(a[i]);
        if (two) {
#pragma unroll
            for (int i = 0; i < 32; ++i) acc += __uint_as_float(b[i]);
        }
    }
    const unsigned long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) sink[threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(slot);
    }
}

int main(int argc, char** argv) {
    const int W = atoi(argv[1]), two = atoi(argv[2]);
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 148 * 8);
    cudaMalloc(&sink, 4096);
    kern<<<148, 32 * W>>>(two, d, sink);
    kern<<<148, 32 * W>>>(two, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    m /= 148;
    const double bytes = (double)W * 32 * 32 * 4 * (two ? 2 : 1) * REPS;
    printf("warps=%d x%d: %.1f clk per round, %.1f B/clk/SM  %s\n", W, two ? 64 : 32, m / REPS, bytes / m,
           cudaGetErrorString(e));
    return 0;
}
