// pool.cu — query pooling, Eq. 2 (Alg. 1 line P:770).
//
//   Q_p[i] = (1/h_i) * sum_{t in block i} Q[t],  h_i = P_q except a ragged last block
//   (its true height, reading R7).
//
// Rounding contract (reading R11): the block sum is accumulated in fp64 in row
// order, divided by h_i in fp64 (IEEE), and rounded ONCE to bf16 with
// round-to-nearest-even (fp64 -> fp32 round-to-odd -> bf16 RNE, which is exact RNE
// because fp32 carries >= 2 extra bits).  HBM-bound: reads Q once (2*N*D bytes per
// head), writes Q_p (2*N_p*D bytes).
#include "common.cuh"
#include "kernels.cuh"

namespace va {

__device__ __forceinline__ __nv_bfloat16 f64_to_bf16_rne(double x) {
    float f = __double2float_rz(x);
    if ((double)f != x) f = __uint_as_float(__float_as_uint(f) | 1u);  // round-to-odd sticky bit
    return __float2bfloat16_rn(f);
}

// One thread = 2 adjacent columns of one pooled row; D/2 threads per pooled row.
template <int D>
__global__ void __launch_bounds__(256) pool_kernel(const __nv_bfloat162* __restrict__ q,
                                                   __nv_bfloat162* __restrict__ qp, int64_t BH, int64_t N,
                                                   int64_t Np, int32_t pq) {
    constexpr int TPR = D / 2;            // threads per pooled row
    constexpr int RPB = 256 / TPR;        // pooled rows per block
    const int64_t prow = (int64_t)blockIdx.x * RPB + threadIdx.x / TPR;  // global pooled row (bh*Np+i)
    const int c2 = threadIdx.x % TPR;
    if (prow >= BH * Np) return;
    const int64_t bh = prow / Np, i = prow % Np;
    const int64_t r0 = i * pq;
    const int64_t r1 = min(N, r0 + (int64_t)pq);
    const __nv_bfloat162* src = q + (bh * N + r0) * TPR + c2;
    double s0 = 0.0, s1 = 0.0;
    int64_t n = r1 - r0;
    int64_t r = 0;
    // 8-deep load batches for memory-level parallelism; adds stay in row order.
    for (; r + 8 <= n; r += 8) {
        __nv_bfloat162 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (r + u) * TPR);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            float2 f = __bfloat1622float2(v[u]);
            s0 += (double)f.x;
            s1 += (double)f.y;
        }
    }
    for (; r < n; ++r) {
        float2 f = __bfloat1622float2(__ldg(src + r * TPR));
        s0 += (double)f.x;
        s1 += (double)f.y;
    }
    const double h = (double)n;
    __nv_bfloat162 out;
    out.x = f64_to_bf16_rne(s0 / h);
    out.y = f64_to_bf16_rne(s1 / h);
    qp[prow * TPR + c2] = out;
}

cudaError_t launch_pool(const void* q, void* qp, int64_t BH, int64_t N, int64_t D, int32_t pq,
                        cudaStream_t st) {
    const int64_t Np = (N + pq - 1) / pq;
    const int64_t rows = BH * Np;
    if (D == 128) {
        const int64_t grid = (rows + 3) / 4;
        pool_kernel<128><<<(unsigned)grid, 256, 0, st>>>((const __nv_bfloat162*)q, (__nv_bfloat162*)qp, BH, N,
                                                         Np, pq);
    } else {
        const int64_t grid = (rows + 7) / 8;
        pool_kernel<64><<<(unsigned)grid, 256, 0, st>>>((const __nv_bfloat162*)q, (__nv_bfloat162*)qp, BH, N,
                                                        Np, pq);
    }
    return cudaGetLastError();
}

}  // namespace va
