// Microbenchmark: tcgen05.mma kind::f16 (bf16, fp32 accumulate) issue-to-completion rate on
// one CTA per SM, M = 128, N in {64, 128, 256}, K = 16 per instruction, A from shared memory
// (SS) or from TMEM (TS), optional concurrent TMA-like smem writes are not modelled.
// Usage: ubench_mma <N> <ts 0/1>
#include "../paper_2603_29494_b200/csrc/common.cuh"
#include <cstdio>
#include <cstdlib>

using namespace va;
constexpr int REPS = 4096;

__global__ void __launch_bounds__(128, 1) kern(int N, int ts, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536 + 65536);
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 65536 + 65536 + 64);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    fence_proxy_async();
    if (warp == 0) tmem_alloc<512>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = *slot;
    unsigned long long t0 = 0, t1 = 0;
    if (warp == 0 && elect_one()) {
        const uint32_t idesc = make_idesc_bf16(128, N, 0, 0);
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
        t0 = clock64();
        for (int r = 0; r < REPS; ++r) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t bd = make_sdesc(b + (kk >> 2) * N * 128 + (kk & 3) * 32, 16, 1024);
                if (ts) {
                    mma_bf16_ts(tm, tm + 256 + kk * 8, bd, idesc, 1u);
                } else {
                    const uint64_t ad = make_sdesc(a + (kk >> 2) * 128 * 128 + (kk & 3) * 32, 16, 1024);
                    mma_bf16_ss(tm, ad, bd, idesc, 1u);
                }
            }
        }
        mma_commit(bar);
        mbar_wait(bar, 0);
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tm);
    }
}

int main(int argc, char** argv) {
    const int N = atoi(argv[1]), ts = atoi(argv[2]);
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    const int smem = 131072 + 128;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<148, 128, smem>>>(N, ts, d);
    kern<<<148, 128, smem>>>(N, ts, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    m /= 148;
    const double per = m / (REPS * 8.0);
    const double floor_ = 128.0 * N / 256.0;
    printf("N=%d %s: %.1f clk/instr (floor %.0f) -> %.0f%% of tensor peak  %s\n", N, ts ? "TS" : "SS", per, floor_,
           100.0 * floor_ / per, cudaGetErrorString(e));
    return 0;
}
