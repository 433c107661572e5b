// Microbenchmark: does TMA tile::gather4 with .multicast::cluster raise the per-SM row-gather
// rate of the sparse attention's K/V path?  (profiles/ubench_r01.md, "What bounds the
// double-buffered kernel": one gather4 per ~29 clk per SM, 17.7 B/clk.)
//
// Each CTA streams ITERS stages of 64 K rows + 64 V rows (256 B each, 32 KB) through an
// S-stage ring; rows are random within a 131072-row head, index lists read from memory
// per stage (sorted ascending, like the attention plan).
//   cs = 1: every CTA gathers its own stage: 64 gather4 per stage per SM.
//   cs = 2: clusters of 2 CTAs consume the SAME row lists; CTA r issues the gather4s of
//           rows [32r, 32r+32) of K and V with ctaMask 0b11, so each SM issues 32
//           gather4 per stage and receives the full 32 KB.  A stage is refilled only when
//           both CTAs' consumers released it (EMPTY count 2: local + remote arrive).
// Usage: ubench_mcast <cs> <stages> <loader warps> [heads in flight (64 MB each)] [hashed rows 0/1]
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
    const int* idx;  // [n_lists][ITERS][64]
    int cs, stages, W, nh, hash;
    unsigned long long* cyc;
};

VA_DEV uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
VA_DEV void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
VA_DEV void arrive_remote(uint64_t* bar, uint32_t rank) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
VA_DEV void gather4_mc(void* dst, const void* desc, uint64_t* bar, int c0, int r0, int r1, int r2, int r3,
                       uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(dst)),
        "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "h"(mask)
        : "memory");
}

__global__ void __launch_bounds__(544, 1) kern(const __grid_constant__ P p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * 32768);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = p.cs == 2 ? cluster_rank() : 0u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], p.cs);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (p.cs == 2) cluster_sync();
    const int list = blockIdx.x / p.cs;  // both CTAs of a cluster read the same rows
    const int* idx = p.idx + (size_t)list * ITERS * ROWS;
    const int head = list % p.nh;
    unsigned long long t0 = clock64();
    if (warp < p.W) {
        // warp w handles row slots [w*R, (w+1)*R) of this CTA's share (K rows, then V rows)
        const int share = 128 / p.cs;        // rows this CTA issues per stage (K + V)
        const int R = share / p.W;
        const int r0 = (int)rank * (64 / p.cs) + 0;  // first K row slot of this CTA
        for (int it = 0; it < ITERS; ++it) {
            const int s = it % S, round = it / S;
            if (lane == 0 && round > 0) mbar_wait(&empty[s], (round - 1) & 1);
            __syncwarp();
            if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&full[s], 32768);
            // slot q in [0, share): K rows first (q < share/2), then V rows
            const int q = warp * R + lane;
            const bool isK = q < share / 2;
            const int rl = r0 + (isK ? q : q - share / 2);  // row within the 64-row tile
            int row = 0;
            if (p.hash) {  // no index load on the critical path; same rows for both CTAs of a cluster
                uint32_t x = (uint32_t)(list * 7919 + it * 131 + rl) * 2654435761u;
                x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
                row = head * 131072 + (int)(x % 131072u);
            } else if (lane < R) {
                row = head * 131072 + __ldg(idx + it * ROWS + rl);
            }
            const int g0 = (4 * lane) & 31;
            const int ra = __shfl_sync(~0u, row, g0), rb = __shfl_sync(~0u, row, g0 + 1);
            const int rc = __shfl_sync(~0u, row, g0 + 2), rd = __shfl_sync(~0u, row, g0 + 3);
            const int rla = __shfl_sync(~0u, rl, g0);
            const bool isKa = __shfl_sync(~0u, (int)isK, g0);
            if (lane < R / 4) {
                uint8_t* d = smem + s * 32768 + (isKa ? 0 : 16384) + rla * 128;
                const void* tm = isKa ? (const void*)&p.tk : (const void*)&p.tv;
                if (p.cs == 2) {
                    gather4_mc(d, tm, &full[s], 0, ra, rb, rc, rd, 3);
                    gather4_mc(d + ROWS * 128, tm, &full[s], 64, ra, rb, rc, rd, 3);
                } else {
                    tma_gather4(d, tm, &full[s], 0, ra, rb, rc, rd);
                    tma_gather4(d + ROWS * 128, tm, &full[s], 64, ra, rb, rc, rd);
                }
            }
        }
    } else if (lane == 0) {
        for (int it = 0; it < ITERS; ++it) {
            const int s = it % S;
            mbar_wait(&full[s], (it / S) & 1);
            mbar_arrive(&empty[s]);
            if (p.cs == 2) arrive_remote(&empty[s], rank ^ 1u);
        }
        p.cyc[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
    if (p.cs == 2) cluster_sync();
}

int main(int argc, char** argv) {
    const int cs = atoi(argv[1]), S = atoi(argv[2]), W = atoi(argv[3]), nh = argc > 4 ? atoi(argv[4]) : 4, hs = argc > 5 ? atoi(argv[5]) : 0;
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int grid = nsm;  // 148, even
    uint8_t *k, *v;
    const long rows_total = 131072L * 4;
    cudaMalloc(&k, rows_total * 256);
    cudaMalloc(&v, rows_total * 256);
    cudaMemset(k, 1, rows_total * 256);
    cudaMemset(v, 2, rows_total * 256);
    const int n_lists = grid / cs;
    std::vector<int> h((size_t)n_lists * ITERS * ROWS);
    std::mt19937 rng(1);
    for (int c = 0; c < n_lists; ++c)
        for (int it = 0; it < ITERS; ++it) {
            int* r = &h[((size_t)c * ITERS + it) * ROWS];
            for (int j = 0; j < ROWS; ++j) r[j] = (int)(rng() % 131072);
            std::sort(r, r + ROWS);
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
    p.idx = di; p.cs = cs; p.stages = S; p.W = W; p.nh = nh; p.hash = hs;
    cudaMalloc(&p.cyc, grid * 8);
    const int smem = S * 32768 + 2 * S * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (cs == 2) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32 * (W + 1));
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, kern, p);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, kern, p);
    cudaEventRecord(b);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> cyc(grid);
    cudaMemcpy(cyc.data(), p.cyc, grid * 8, cudaMemcpyDeviceToHost);
    double mc = 0;
    for (auto c : cyc) mc += c;
    mc /= grid;
    const double bytes = (double)grid * ITERS * 32768;  // bytes delivered into shared memory
    printf("nh=%d cs=%d S=%d W=%d: %.3f ms  delivered %.2f TB/s  %.1f B/clk/SM  %.0f clk/stage/CTA  %s\n", nh, cs, S, W, ms,
           bytes / ms / 1e9, bytes / nsm / mc * nsm / grid, mc / ITERS, cudaGetErrorString(err));
    return 0;
}
