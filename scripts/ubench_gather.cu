// Microbenchmark: per-SM row-gather throughput into shared memory (the sparse attention's
// K/V path).  Each CTA streams ITERS stages of 64 K rows + 64 V rows (256 B each, 32 KB
// per stage) from random rows of a working set, through an S-stage ring.
//   mode 0: TMA tile::gather4 (4 warps, lanes 0-7, 2 x 128-B column blocks)
//   mode 1: cp.async 16 B per lane (4 warps x 32 lanes), cp.async.mbarrier.arrive.noinc
// Usage: ubench_gather <mode> <stages> <ctas_per_sm> <span_rows> <sorted 0/1>
#include "../paper_2603_29494_b200/csrc/common.cuh"
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

using namespace va;
constexpr int ITERS = 2000;
constexpr int ROWS = 64;

PFN_cuTensorMapEncodeTiled_v12000 enc() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

struct P {
    CUtensorMap tk, tv;
    const uint8_t* k;
    const uint8_t* v;
    const int* idx;  // [grid][ITERS][64]
    int mode, stages, W, hash, span;
    unsigned long long* cyc;
};

VA_DEV void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
VA_DEV void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(544, 1) kern(const __grid_constant__ P p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * 32768);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], p.mode == 0 ? p.W : 32 * p.W);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int* idx = p.idx + (size_t)blockIdx.x * ITERS * ROWS;
    unsigned long long t0 = clock64();
    if (warp < p.W) {
        const int R = 128 / p.W;             // rows per warp (K rows first, then V rows)
        const int r0 = warp * R;
        const bool isK = r0 < 64;
        const int rt = r0 & 63;              // first row within the 64-row tile
        for (int it = 0; it < ITERS; ++it) {
            const int s = it % S, round = it / S;
            if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
            int row = 0;
            if (p.hash) {  // no index load on the critical path
                uint32_t x = (uint32_t)(blockIdx.x * 7919 + it * 131 + rt + lane) * 2654435761u;
                x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
                row = (int)((blockIdx.x / 37) % 4) * 131072 + (int)(x % (uint32_t)p.span);
            } else row = lane < R ? __ldg(idx + it * ROWS + rt + lane) : 0;
            uint8_t* dst = smem + s * 32768 + (isK ? 0 : 16384);
            if (p.mode == 0) {
                if (lane == 0) mbar_arrive_expect_tx(&full[s], R * 256);
                const int q0 = (4 * lane) & 31;
                const int ra = __shfl_sync(~0u, row, q0), rb = __shfl_sync(~0u, row, q0 + 1);
                const int rc = __shfl_sync(~0u, row, q0 + 2), rd = __shfl_sync(~0u, row, q0 + 3);
                if (lane < R / 4) {
                    uint8_t* d = dst + (rt + 4 * lane) * 128;
                    tma_gather4(d, isK ? &p.tk : &p.tv, &full[s], 0, ra, rb, rc, rd);
                    tma_gather4(d + ROWS * 128, isK ? &p.tk : &p.tv, &full[s], 64, ra, rb, rc, rd);
                }
            } else {
                const uint8_t* base = isK ? p.k : p.v;
                for (int u = 0; u < R / 2; ++u) {
                    const int rl = 2 * u + (lane >> 4);
                    const int r = __shfl_sync(~0u, row, rl);
                    const int pc = lane & 15;
                    const int cb = pc >> 3, c16 = pc & 7;
                    const int rr = rt + rl;
                    const uint32_t d = smem_u32(dst + cb * ROWS * 128 + rr * 128 + ((c16 ^ (rr & 7)) << 4));
                    cp_async16(d, base + (size_t)r * 256 + pc * 16);
                }
                cp_async_arrive(&full[s]);
            }
        }
    } else if (lane == 0) {
        for (int it = 0; it < ITERS; ++it) {
            const int s = it % S;
            mbar_wait(&full[s], (it / S) & 1);
            mbar_arrive(&empty[s]);
        }
        p.cyc[blockIdx.x] = clock64() - t0;
    }
}

int main(int argc, char** argv) {
    const int mode = atoi(argv[1]), S = atoi(argv[2]), cps = atoi(argv[3]), W = argc > 6 ? atoi(argv[6]) : 4;
    const long span = atol(argv[4]);
    const int sorted = atoi(argv[5]);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int grid = nsm * cps;
    uint8_t *k, *v;
    const long rows_total = 131072 * 4;
    cudaMalloc(&k, rows_total * 256);
    cudaMalloc(&v, rows_total * 256);
    cudaMemset(k, 1, rows_total * 256);
    cudaMemset(v, 2, rows_total * 256);
    std::vector<int> h((size_t)grid * ITERS * ROWS);
    std::mt19937 rng(1);
    for (int c = 0; c < grid; ++c) {
        // each group of 8 CTAs works on its own head-sized span (like head-major items)
        const long base = (long)((c / 37) % 4) * 131072;
        for (int it = 0; it < ITERS; ++it) {
            int* r = &h[((size_t)c * ITERS + it) * ROWS];
            for (int j = 0; j < ROWS; ++j) r[j] = (int)(base + rng() % span);
            if (sorted) std::sort(r, r + ROWS);
        }
    }
    int* di;
    cudaMalloc(&di, h.size() * 4);
    cudaMemcpy(di, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    P p{};
    auto e = enc();
    for (int t = 0; t < 2; ++t) {
        cuuint64_t dims[2] = {128, (cuuint64_t)rows_total};
        cuuint64_t strides[1] = {256};
        cuuint32_t box[2] = {64, 1};
        cuuint32_t es[2] = {1, 1};
        e(t ? &p.tv : &p.tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, t ? v : k, dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    p.k = k; p.v = v; p.idx = di; p.mode = mode; p.stages = S; p.W = W; p.hash = argc > 7 ? atoi(argv[7]) : 0; p.span = (int)span;
    cudaMalloc(&p.cyc, grid * 8);
    const int smem = S * 32768 + 2 * S * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    kern<<<grid, 32 * (W + 1), smem>>>(p);
    cudaEventRecord(a);
    kern<<<grid, 32 * (W + 1), smem>>>(p);
    cudaEventRecord(b);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> cyc(grid);
    cudaMemcpy(cyc.data(), p.cyc, grid * 8, cudaMemcpyDeviceToHost);
    double mc = 0;
    for (auto c : cyc) mc += c;
    mc /= grid;
    const double bytes = (double)grid * ITERS * 32768;
    printf("W=%d mode=%d S=%d cps=%d span=%ld sorted=%d: %.3f ms  %.2f TB/s  %.1f B/clk/SM  %.0f clk/stage/CTA  %s\n", W, mode, S,
           cps, span, sorted, ms, bytes / ms / 1e9, bytes / nsm / (mc), mc / ITERS, cudaGetErrorString(err));
    return 0;
}
