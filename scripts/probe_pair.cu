// Probe of tcgen05 CTA-pair (cta_group::2) semantics before the pair attention kernel:
//   S = A B^T with M = 256 (A rows 0-127 in CTA 0's smem, 128-255 in CTA 1's), N = 128
//   (which CTA holds which half of B?), K = 128, SS; then O = P V with P (bf16) from each
//   CTA's TMEM (TS) and V split along N (D columns).  Prints max |err| against a host
//   reference for each hypothesis, plus the issue rate of back-to-back pair MMAs.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o probe_pair probe_pair.cu
#include "../paper_2603_29494_b200/csrc/common.cuh"
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

using namespace va;

VA_DEV uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
VA_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
VA_DEV void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
VA_DEV void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
VA_DEV void commit2(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
// SW128 K-major byte offset of (row r, element k) in a [rows x 64] bf16 block
__host__ __device__ inline uint32_t sw128(int r, int k) {
    return (r >> 3) * 1024 + (r & 7) * 128 + ((((k * 2) >> 4) ^ (r & 7)) << 4) + ((k * 2) & 15);
}


VA_DEV uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
VA_DEV void gather4_pair(uint32_t dst, const void* desc, uint32_t bar_cluster, int c0, int r0, int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.cta_group::2"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
        "l"(desc), "r"(bar_cluster), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}
VA_DEV void remote_arrive(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
VA_DEV bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Each CTA gathers 8 rows (rank-dependent) x 128 cols into its own smem; both CTAs' TMAs
// complete on the LEADER's barrier (count 2: leader expect_tx + peer remote arrive).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1)
    probe_gather(const __grid_constant__ CUtensorMap tm, const __nv_bfloat16* K, int* bad) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8192);
    const uint32_t rank = cluster_rank();
    if (threadIdx.x == 0) {
        mbar_init(bar, 2);
        fence_barrier_init();
    }
    cluster_sync_all();
    const uint32_t lbar = mapa_rank(smem_u32(bar), 0);
    const int rows[8] = {3 + 100 * (int)rank, 17, 250, 1023, 5 + (int)rank, 600, 64, 65};
    if (threadIdx.x == 0) {
        if (rank == 0) mbar_arrive_expect_tx(bar, 2 * 2 * 8 * 128);
        for (int cb = 0; cb < 2; ++cb)
            for (int g = 0; g < 2; ++g)
                gather4_pair(smem_u32(smem + cb * 8 * 128 + g * 512), &tm, lbar, cb * 64, rows[4 * g], rows[4 * g + 1],
                             rows[4 * g + 2], rows[4 * g + 3]);
        if (rank == 1) remote_arrive(lbar);
        if (rank == 0) while (!mbar_try_wait_cluster(bar, 0)) {}
    }
    cluster_sync_all();
    for (int x = threadIdx.x; x < 8 * 128; x += 64) {
        const int i = x / 128, k = x % 128;
        const __nv_bfloat16 got = *reinterpret_cast<__nv_bfloat16*>(smem + (k >> 6) * 8 * 128 + sw128(i, k & 63));
        if (__bfloat162float(got) != __bfloat162float(K[rows[i] * 128 + k])) atomicAdd(bad, 1);
    }
}

// A [256 x 128], B [128 x 128] (rows = N index), V [128 keys x 128 cols]; outputs S [256 x 128], O [256 x 128]
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(const __nv_bfloat16* A, const __nv_bfloat16* B, const __nv_bfloat16* V, float* S, float* O,
          long long* clk, int bhalf_swap) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;               // 2 col blocks x [128 x 64] = 32 KB
    uint8_t* sB = smem + 32768;       // 2 col blocks x [64 x 64]  = 16 KB
    uint8_t* sV = smem + 49152;       // [128 keys x 64 cols] MN-major = 16 KB
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 65536 + 64);
    const uint32_t rank = cluster_rank();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int brank = bhalf_swap ? 1 - (int)rank : (int)rank;
    for (int x = threadIdx.x; x < 128 * 128; x += 128) {
        const int r = x / 128, k = x % 128;
        *reinterpret_cast<__nv_bfloat16*>(sA + (k >> 6) * 16384 + sw128(r, k & 63)) = A[(128 * rank + r) * 128 + k];
    }
    for (int x = threadIdx.x; x < 64 * 128; x += 128) {
        const int r = x / 128, k = x % 128;
        *reinterpret_cast<__nv_bfloat16*>(sB + (k >> 6) * 8192 + sw128(r, k & 63)) = B[(64 * brank + r) * 128 + k];
    }
    for (int x = threadIdx.x; x < 128 * 64; x += 128) {
        const int j = x / 64, n = x % 64;  // key j, column 64*rank + n
        *reinterpret_cast<__nv_bfloat16*>(sV + sw128(j, n)) = V[j * 128 + 64 * rank + n];
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&bar[2], 1);
        fence_barrier_init();
    }
    fence_proxy_async();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tm = *slot;
    const uint32_t idS = make_idesc_bf16(256, 128, 0, 0), idPV = make_idesc_bf16(256, 128, 0, 1);
    if (rank == 0 && warp == 1 && elect_one()) {
        for (int kk = 0; kk < 8; ++kk) {
            const uint64_t ad = make_sdesc(smem_u32(sA) + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = make_sdesc(smem_u32(sB) + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
            mma2_ss(tm + 128, ad, bd, idS, kk > 0);
        }
        commit2(&bar[0]);
    }
    mbar_wait(&bar[0], 0);
    tc_fence_after();
    // S rows of this CTA: TMEM lane = row within the CTA's half
    const int row = 32 * warp + lane;
    uint32_t pk[32];
    for (int g = 0; g < 4; ++g) {
        uint32_t v[32];
        tmem_ld32(tm + ((uint32_t)(32 * warp) << 16) + 128 + 32 * g, v);
        tmem_ld_wait();
        for (int t = 0; t < 32; ++t) S[(128 * rank + row) * 128 + 32 * g + t] = __uint_as_float(v[t]);
        for (int t = 0; t < 32; t += 2)
            pk[16 * (g & 1) + t / 2] = pack_bf16x2(__uint_as_float(v[t]) * 0.0625f, __uint_as_float(v[t + 1]) * 0.0625f);
        if (g & 1) tmem_st32(tm + ((uint32_t)(32 * warp) << 16) + 256 + 32 * (g >> 1), pk);
    }
    tmem_st_wait();
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (rank == 0 && warp == 1 && elect_one()) {
        for (int kk = 0; kk < 8; ++kk) {
            const uint64_t bd = make_sdesc(smem_u32(sV) + kk * 16 * 128, 128 * 128, 1024);
            mma2_ts(tm, tm + 256 + 8 * kk, bd, idPV, kk > 0);
        }
        commit2(&bar[1]);
    }
    mbar_wait(&bar[1], 0);
    tc_fence_after();
    for (int g = 0; g < 4; ++g) {
        uint32_t v[32];
        tmem_ld32(tm + ((uint32_t)(32 * warp) << 16) + 32 * g, v);
        tmem_ld_wait();
        for (int t = 0; t < 32; ++t) O[(128 * rank + row) * 128 + 32 * g + t] = __uint_as_float(v[t]);
    }
    // issue rate: 512 back-to-back pair MMAs, SS (S shape) then TS (PV shape)
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (rank == 0 && warp == 1 && elect_one()) {
        const uint64_t ad = make_sdesc(smem_u32(sA), 16, 1024), bd = make_sdesc(smem_u32(sB), 16, 1024);
        const uint64_t vd = make_sdesc(smem_u32(sV), 128 * 128, 1024);
        long long t0 = clock64();
        for (int i = 0; i < 512; ++i) mma2_ss(tm + 128, ad, bd, idS, 1);
        commit2(&bar[2]);
        mbar_wait(&bar[2], 0);
        long long t1 = clock64();
        for (int i = 0; i < 512; ++i) mma2_ts(tm, tm + 256, vd, idPV, 1);
        commit2(&bar[2]);
        mbar_wait(&bar[2], 1);
        long long t2 = clock64();
        clk[0] = t1 - t0;
        clk[1] = t2 - t1;
    } else if (warp != 1) {
    }
    if (rank == 1 && threadIdx.x == 0) {
        mbar_wait(&bar[2], 0);
        mbar_wait(&bar[2], 1);
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

static float bf(float x) {  // round to bf16
    uint32_t u;
    memcpy(&u, &x, 4);
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000u;
    float y;
    memcpy(&y, &u, 4);
    return y;
}

int main(int argc, char** argv) {
    const int swap = argc > 1 ? atoi(argv[1]) : 0;
    std::vector<float> A(256 * 128), B(128 * 128), V(128 * 128);
    std::vector<__nv_bfloat16> Ah(A.size()), Bh(B.size()), Vh(V.size());
    srand(1);
    auto rnd = [] { return (float)((rand() % 17) - 8) / 8.f; };
    for (size_t i = 0; i < A.size(); ++i) { A[i] = bf(rnd()); Ah[i] = __float2bfloat16(A[i]); }
    for (size_t i = 0; i < B.size(); ++i) { B[i] = bf(rnd()); Bh[i] = __float2bfloat16(B[i]); }
    for (size_t i = 0; i < V.size(); ++i) { V[i] = bf(rnd()); Vh[i] = __float2bfloat16(V[i]); }
    __nv_bfloat16 *dA, *dB, *dV;
    float *dS, *dO;
    long long* dc;
    cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dV, V.size() * 2);
    cudaMalloc(&dS, 256 * 128 * 4); cudaMalloc(&dO, 256 * 128 * 4); cudaMalloc(&dc, 16);
    cudaMemcpy(dA, Ah.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bh.data(), B.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dV, Vh.data(), V.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    probe<<<2, 128, 70000>>>(dA, dB, dV, dS, dO, dc, swap);
    cudaError_t e = cudaDeviceSynchronize();
    printf("swap=%d launch: %s\n", swap, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<float> S(256 * 128), O(256 * 128);
    long long c[2];
    cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
    // hypothesis: S[m][n] = sum_k A[m][k] B[n][k] with B row n held by CTA n/64 (swap=0)
    double es = 0, eo = 0;
    std::vector<float> P(256 * 128);
    for (int m = 0; m < 256; ++m)
        for (int n = 0; n < 128; ++n) {
            double s = 0;
            for (int k = 0; k < 128; ++k) s += (double)A[m * 128 + k] * B[n * 128 + k];
            es = fmax(es, fabs(s - S[m * 128 + n]));
            P[m * 128 + n] = bf((float)s * 0.0625f);
        }
    for (int m = 0; m < 256; ++m)
        for (int n = 0; n < 128; ++n) {
            double s = 0;
            for (int j = 0; j < 128; ++j) s += (double)P[m * 128 + j] * V[j * 128 + n];
            eo = fmax(eo, fabs(s - O[m * 128 + n]));
        }
    printf("S max err %.4g  (S[0][0]=%g S[0][64]=%g S[200][100]=%g)\n", es, S[0], S[64], S[200 * 128 + 100]);
    printf("O max err %.4g\n", eo);
    printf("512 pair MMAs M256 N128 K16: SS %.1f clk/instr, TS %.1f clk/instr\n", c[0] / 512.0, c[1] / 512.0);
    {   // gather4 with .cta_group::2 completing on the leader's barrier
        typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        std::vector<__nv_bfloat16> Kh(1024 * 128);
        for (size_t i = 0; i < Kh.size(); ++i) Kh[i] = __float2bfloat16((float)(i % 251));
        __nv_bfloat16* dK;
        int* dbad;
        cudaMalloc(&dK, Kh.size() * 2);
        cudaMalloc(&dbad, 4);
        cudaMemset(dbad, 0, 4);
        cudaMemcpy(dK, Kh.data(), Kh.size() * 2, cudaMemcpyHostToDevice);
        CUtensorMap tm;
        cuuint64_t dims[2] = {128, 1024}, strides[1] = {256};
        cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
        CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dK, dims, strides, box, es,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaFuncSetAttribute(probe_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 9216);
        probe_gather<<<2, 64, 9216>>>(tm, dK, dbad);
        cudaError_t e2 = cudaDeviceSynchronize();
        int bad = -1;
        cudaMemcpy(&bad, dbad, 4, cudaMemcpyDeviceToHost);
        printf("gather4.cta_group::2 -> leader barrier: encode %d, launch %s, mismatches %d\n", (int)r,
               cudaGetErrorString(e2), bad);
    }
    return 0;
}
