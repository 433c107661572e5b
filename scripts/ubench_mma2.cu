// Microbenchmark: tcgen05.mma issue patterns for the sparse attention S = Q K^T step
// (M = 128, K = 16 per instruction, bf16, one CTA per SM).
//   mode 0: one accumulator, A (Q slice) and B (K slice) from SMEM          (the S chain)
//   mode 1: two accumulators interleaved per K-step, different A, same B   (tile 0 / tile 1)
//   mode 2: two accumulators, same A, different B, no collector hint      (chunk j / j+1)
//   mode 3: as 2 with .collector::a::fill then .collector::a::lastuse      (A read once)
//   mode 4: A from TMEM, one accumulator                                    (TS reference)
//   mode 5: two accumulators, blocked: 8 K-steps into acc 0, then 8 into acc 1
//   mode 6: A from TMEM, two accumulators interleaved, same B                (PV of 2 tiles)
//   mode 7: A from TMEM, two accumulators blocked
// Usage: ubench_mma2 <N> <mode>
#include "../paper_2603_29494_b200/csrc/common.cuh"
#include <cstdio>
#include <cstdlib>

using namespace va;
constexpr int REPS = 2048;

VA_DEV void mma_ss_fill(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, 1;\n" ::"r"(d), "l"(a),
                 "l"(b), "r"(idesc)
                 : "memory");
}
VA_DEV void mma_ss_lastuse(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, 1;\n" ::"r"(d), "l"(a),
                 "l"(b), "r"(idesc)
                 : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) kern(int N, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 4 * 32768);
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 4 * 32768 + 64);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 4 * 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
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
    if (warp == 0 && elect_one()) {
        const uint32_t idesc = make_idesc_bf16(128, N, 0, 0);
        const uint32_t a0 = smem_u32(smem), a1 = smem_u32(smem + 32768);
        const uint32_t b0 = smem_u32(smem + 65536), b1 = smem_u32(smem + 65536 + 32768);
        uint64_t A0[8], A1[8], B0[8], B1[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const uint32_t ao = (kk >> 2) * 128 * 128 + (kk & 3) * 32;
            const uint32_t bo = (kk >> 2) * N * 128 + (kk & 3) * 32;
            A0[kk] = make_sdesc(a0 + ao, 16, 1024);
            A1[kk] = make_sdesc(a1 + ao, 16, 1024);
            B0[kk] = make_sdesc(b0 + bo, 16, 1024);
            B1[kk] = make_sdesc(b1 + bo, 16, 1024);
        }
        constexpr int per = (MODE == 0 || MODE == 4) ? 8 : 16;
        const unsigned long long t0 = clock64();
        for (int r = 0; r < REPS; ++r) {
            if constexpr (MODE == 5) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_bf16_ss(tm, A0[kk], B0[kk], idesc, 1u);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_bf16_ss(tm + 256, A1[kk], B0[kk], idesc, 1u);
            } else if constexpr (MODE == 7) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_bf16_ts(tm, tm + 256 + kk * 8, B0[kk], idesc, 1u);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma_bf16_ts(tm + 128, tm + 384 + kk * 8, B0[kk], idesc, 1u);
            } else {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    if constexpr (MODE == 0) {
                        mma_bf16_ss(tm, A0[kk], B0[kk], idesc, 1u);
                    } else if constexpr (MODE == 1) {
                        mma_bf16_ss(tm, A0[kk], B0[kk], idesc, 1u);
                        mma_bf16_ss(tm + 256, A1[kk], B0[kk], idesc, 1u);
                    } else if constexpr (MODE == 2) {
                        mma_bf16_ss(tm, A0[kk], B0[kk], idesc, 1u);
                        mma_bf16_ss(tm + 256, A0[kk], B1[kk], idesc, 1u);
                    } else if constexpr (MODE == 3) {
                        mma_ss_fill(tm, A0[kk], B0[kk], idesc);
                        mma_ss_lastuse(tm + 256, A0[kk], B1[kk], idesc);
                    } else if constexpr (MODE == 4) {
                        mma_bf16_ts(tm, tm + 256 + kk * 8, B0[kk], idesc, 1u);
                    } else if constexpr (MODE == 6) {
                        mma_bf16_ts(tm, tm + 256 + kk * 8, B0[kk], idesc, 1u);
                        mma_bf16_ts(tm + 128, tm + 384 + kk * 8, B0[kk], idesc, 1u);
                    }
                }
            }
        }
        mma_commit(bar);
        mbar_wait(bar, 0);
        const unsigned long long t1 = clock64();
        out[blockIdx.x] = (t1 - t0);
        out[148 + blockIdx.x] = (unsigned long long)REPS * per;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tm);
    }
}

template <int MODE>
void run(int N, unsigned long long* d) {
    const int smem = 4 * 32768 + 128;
    cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<MODE><<<148, 128, smem>>>(N, d);
    kern<MODE><<<148, 128, smem>>>(N, d);
}

int main(int argc, char** argv) {
    const int N = atoi(argv[1]), mode = atoi(argv[2]);
    unsigned long long* d;
    cudaMalloc(&d, 2 * 148 * 8);
    switch (mode) {
        case 0: run<0>(N, d); break;
        case 1: run<1>(N, d); break;
        case 2: run<2>(N, d); break;
        case 3: run<3>(N, d); break;
        case 4: run<4>(N, d); break;
        case 5: run<5>(N, d); break;
        case 6: run<6>(N, d); break;
        default: run<7>(N, d); break;
    }
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[2 * 148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    m /= 148;
    const double per = m / (double)h[148];
    const double floor_ = 128.0 * N / 256.0;
    printf("N=%d mode %d: %.1f clk/instr (floor %.0f) -> %.0f%% of tensor peak  %s\n", N, mode, per, floor_,
           100.0 * floor_ / per, cudaGetErrorString(e));
    return 0;
}
