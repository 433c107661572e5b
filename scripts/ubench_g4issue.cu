// Microbenchmark: per-warp issue cost of TMA tile::gather4 (the sparse attention's K/V path).
// Each warp streams ITERS batches of 64 random rows x 256 B (32 gather4 of 4 rows x 128 B)
// into two 16 KB buffers (double-buffered, mbarrier complete_tx) and reports clk per gather4
// per warp and the SM's delivered B/clk.
//   variant 0: waterfall -- lanes 0-15 issue with their own coordinates (attn_db.cu loader)
//   variant 1: whole warp shuffles each row quad (uniform source lane), lane 0 issues
//   variant 2: rows staged in shared memory, lane 0 reads each quad (ld.shared.v4) and issues
//   variant 3: as 1, but elect.sync picks the issuing lane
//   mma (argv 4): 0 none; 1 one extra warp issues SS tcgen05.mma M=128 N=64 back to back (the
//   attention's S = Q K^T shape, smem-read-bound) while the gathers run; 2 TS N=128 (A in TMEM);
//   3 SS N=128
//   busy (argv 5): extra warps running a softmax-like ex2/FFMA2 loop (issue-slot competition)
// Usage: ubench_g4issue <variant> <warps per CTA> <span rows> [mma] [busy warps]
#include "../paper_2603_29494_b200/csrc/common.cuh"
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>

using namespace va;
constexpr int ITERS = 1000;

PFN_cuTensorMapEncodeTiled_v12000 enc() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

struct P {
    CUtensorMap tk;
    const int* idx;  // [grid*W][ITERS][64]
    int variant, W, mma, busy;
    unsigned long long* cyc;
    unsigned long long* mma_count;
};

template <int VAR>
__device__ void run(const P& p, uint8_t* smem, uint64_t* bars, int* srows) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* buf = smem + warp * 32768;
    uint64_t* bar = bars + 2 * warp;
    const int* idx = p.idx + ((size_t)blockIdx.x * p.W + warp) * ITERS * 64;
    int* sr = srows + warp * 64;
    int r0n = idx[lane], r1n = idx[32 + lane];
    for (int it = 0; it < ITERS; ++it) {
        const int b = it & 1;
        const int r0 = r0n, r1 = r1n;
        if (it + 1 < ITERS) { r0n = idx[(it + 1) * 64 + lane]; r1n = idx[(it + 1) * 64 + 32 + lane]; }
        if (it >= 2 && lane == 0) mbar_wait(&bar[b], ((it >> 1) - 1) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&bar[b], 16384);
        uint8_t* dst = buf + b * 16384;
        if constexpr (VAR == 0) {
            const int q0 = (4 * lane) & 31;
            const int a0 = __shfl_sync(~0u, r0, q0), a1 = __shfl_sync(~0u, r0, q0 + 1);
            const int a2 = __shfl_sync(~0u, r0, q0 + 2), a3 = __shfl_sync(~0u, r0, q0 + 3);
            const int b0 = __shfl_sync(~0u, r1, q0), b1 = __shfl_sync(~0u, r1, q0 + 1);
            const int b2 = __shfl_sync(~0u, r1, q0 + 2), b3 = __shfl_sync(~0u, r1, q0 + 3);
            const bool lo = lane < 8;
            if (lane < 16) {
                uint8_t* d = dst + 4 * lane * 128;
                for (int cb = 0; cb < 2; ++cb)
                    tma_gather4(d + cb * 64 * 128, &p.tk, &bar[b], cb * 64, lo ? a0 : b0, lo ? a1 : b1, lo ? a2 : b2,
                                lo ? a3 : b3);
            }
        } else if constexpr (VAR == 1 || VAR == 3) {
#pragma unroll
            for (int g = 0; g < 16; ++g) {
                const int src = g < 8 ? r0 : r1;
                const int x0 = __shfl_sync(~0u, src, (4 * g) & 31), x1 = __shfl_sync(~0u, src, (4 * g + 1) & 31);
                const int x2 = __shfl_sync(~0u, src, (4 * g + 2) & 31), x3 = __shfl_sync(~0u, src, (4 * g + 3) & 31);
                const bool go = VAR == 1 ? lane == 0 : elect_one();
                if (go) {
#pragma unroll
                    for (int cb = 0; cb < 2; ++cb)
                        tma_gather4(dst + g * 4 * 128 + cb * 64 * 128, &p.tk, &bar[b], cb * 64, x0, x1, x2, x3);
                }
                __syncwarp();
            }
        } else {
            sr[lane] = r0;
            sr[32 + lane] = r1;
            __syncwarp();
            if (lane == 0) {
#pragma unroll
                for (int g = 0; g < 16; ++g) {
                    const int4 x = reinterpret_cast<const int4*>(sr)[g];
#pragma unroll
                    for (int cb = 0; cb < 2; ++cb)
                        tma_gather4(dst + g * 4 * 128 + cb * 64 * 128, &p.tk, &bar[b], cb * 64, x.x, x.y, x.z, x.w);
                }
            }
            __syncwarp();
        }
    }
    if (lane == 0) {
        mbar_wait(&bar[(ITERS - 2) & 1], ((ITERS - 2) >> 1) & 1);
        mbar_wait(&bar[(ITERS - 1) & 1], ((ITERS - 1) >> 1) & 1);
    }
}

__global__ void __launch_bounds__(1024, 1) kern(const __grid_constant__ P p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int W = p.W;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + W * 32768);
    int* srows = reinterpret_cast<int*>(bars + 2 * W + 1);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2 * W + 1; ++i) mbar_init(&bars[i], 1);
        fence_barrier_init();
    }
    volatile int* done = reinterpret_cast<volatile int*>(srows + 64 * W);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(srows + 64 * W + 4);
    if (threadIdx.x == 0) *done = 0;
    const int warp = threadIdx.x >> 5;
    if (p.mma && warp == W) tmem_alloc<512>(tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    unsigned long long t0 = clock64();
    if (warp < W) {
        switch (p.variant) {
            case 0: run<0>(p, smem, bars, srows); break;
            case 1: run<1>(p, smem, bars, srows); break;
            case 2: run<2>(p, smem, bars, srows); break;
            default: run<3>(p, smem, bars, srows); break;
        }
        __syncwarp();
        if ((threadIdx.x & 31) == 0) atomicAdd((int*)done, 1);
    } else if (warp > W || (warp == W && !p.mma)) {
        // softmax-like issue load: 64 ex2 + 32 FFMA2 + 32 F2FP per "chunk" per lane
        float x = threadIdx.x * 1e-3f, acc = 0.f;
        while (*done < W) {
#pragma unroll 8
            for (int i = 0; i < 64; ++i) {
                const float e = ex2(x - (float)i * 0.01f);
                acc = fmaf(e, 0.5f, acc);
            }
        }
        if (acc == 12345.f) p.cyc[0] = 1;
    } else if (elect_one()) {
        // background tensor-core traffic on the same SM: operands point into the gather buffers
        const uint32_t tm = *tslot;
        const int N = p.mma == 1 ? 64 : 128;
        const uint32_t idesc = make_idesc_bf16(128, N, 0, 0);
        const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 16384);
        unsigned long long n = 0;
        while (*done < W) {
            for (int r = 0; r < 16; ++r) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t bd = make_sdesc(b0 + (kk & 3) * 32, 16, 1024);
                    if (p.mma == 2) mma_bf16_ts(tm, tm + 256 + kk * 8, bd, idesc, 1u);
                    else mma_bf16_ss(tm, make_sdesc(a0 + (kk & 3) * 32, 16, 1024), bd, idesc, 1u);
                }
            }
            n += 128;
            mma_commit(&bars[2 * W]);
            mbar_wait(&bars[2 * W], (uint32_t)((n / 128 - 1) & 1));
        }
        p.mma_count[blockIdx.x] = n;
    }
    __syncthreads();
    if (threadIdx.x == 0) p.cyc[blockIdx.x] = clock64() - t0;
    if (p.mma && warp == W) {
        tc_fence_after();
        tmem_dealloc<512>(*tslot);
    }
}

int main(int argc, char** argv) {
    const int var = atoi(argv[1]), W = atoi(argv[2]);
    const long span = atol(argv[3]);
    const int mma = argc > 4 ? atoi(argv[4]) : 0;
    const int busy = argc > 5 ? atoi(argv[5]) : 0;
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int grid = nsm;
    uint8_t* k;
    const long rows_total = 131072 * 4;
    cudaMalloc(&k, rows_total * 256);
    cudaMemset(k, 1, rows_total * 256);
    std::vector<int> h((size_t)grid * W * ITERS * 64);
    std::mt19937 rng(1);
    for (size_t c = 0; c < h.size() / 64; ++c) {
        const long base = (long)((c / (37 * W)) % 4) * 131072;
        for (int j = 0; j < 64; ++j) h[c * 64 + j] = (int)(base + rng() % span);
    }
    int* di;
    cudaMalloc(&di, h.size() * 4);
    cudaMemcpy(di, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    P p{};
    auto e = enc();
    cuuint64_t dims[2] = {128, (cuuint64_t)rows_total};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, 1};
    cuuint32_t es[2] = {1, 1};
    e(&p.tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, k, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    p.idx = di; p.variant = var; p.W = W; p.mma = mma; p.busy = busy;
    cudaMalloc(&p.cyc, grid * 8);
    cudaMalloc(&p.mma_count, grid * 8);
    cudaMemset(p.mma_count, 0, grid * 8);
    const int smem = W * 32768 + (2 * W + 1) * 8 + W * 256 + 16;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<grid, 32 * (W + (mma ? 1 : 0) + busy), smem>>>(p);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<grid, 32 * (W + (mma ? 1 : 0) + busy), smem>>>(p);
    cudaEventRecord(b);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> cyc(grid);
    cudaMemcpy(cyc.data(), p.cyc, grid * 8, cudaMemcpyDeviceToHost);
    double mc = 0;
    for (auto c : cyc) mc += c;
    mc /= grid;
    const double g4 = (double)ITERS * 32;  // per warp
    std::vector<unsigned long long> mcnt(grid);
    cudaMemcpy(mcnt.data(), p.mma_count, grid * 8, cudaMemcpyDeviceToHost);
    double mm = 0;
    for (auto c : mcnt) mm += c;
    mm /= grid;
    printf("busy=%d variant=%d W=%d span=%ld mma=%d: %.3f ms  %.1f clk/gather4/warp  %.1f B/clk/SM  %.2f TB/s  mma %.1f clk/instr  %s\n",
           busy, var, W, span, mma, ms, mc / g4, g4 * W * 512 / mc, (double)grid * W * g4 * 512 / ms / 1e9,
           mm > 0 ? mc / mm : 0.0, cudaGetErrorString(err));
    return 0;
}
