// naive.cu — the paper's NAIVE materialise-then-filter selection (Fig. 5
// P:281-286), built as the comparison baseline for TilingSelect.
//
// The pooled score map S_p = Q_p K^T (raw fp32 accumulators, the same tcgen05 GEMM as the
// fused path, EPI_SCORES) is written to HBM ([R, N], R = B*Hq*N_p), then filtered row by row:
//   minS  (Eq. 3): m = max_j acc; keep acc >= m - alpha/scale  -> identical
//         decisions to the fused MINS_EXACT (same accumulators, same fp32 threshold).
//   topP: A = softmax(scale * acc) over the visible keys; the keys
//         sorted by descending probability (CUB segmented radix sort, stable: ties keep the
//         lowest index first, reading R12); the smallest prefix with cumulative mass >= p,
//         keys of zero probability never taken.
// Both write the selection bitmask of the fused path (1 bit per key, row stride
// words_per_row) and per-row counts, so offsets and indices come from the same scan and
// emit kernels (compact.cu).  Causal: keys j > L_i are excluded (reading R5).
#include "common.cuh"
#include "kernels.cuh"

#include <cub/cub.cuh>
#include <math.h>
#include <algorithm>

namespace va {

namespace {

constexpr int kRowThreads = 256;

VA_DEV int64_t vis_end(int64_t row, int64_t Np, int64_t N, int32_t pq, int32_t causal) {
    const int64_t i = row % Np;
    return causal ? min(N, (i + 1) * (int64_t)pq) : N;
}

VA_DEV float block_max(float v, float* sh) {
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    v = lane < kRowThreads / 32 ? sh[lane] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    return v;
}

VA_DEV double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    v = lane < kRowThreads / 32 ? sh[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    return v;
}

// Row statistics of the materialised map: max of the raw accumulators over the visible
// keys, and (topP) Z = sum_j exp2((acc_j - max) * scale*log2e) (fp32 terms, fp64 sum).
// Rows are read with 16-B loads when N % 4 == 0 (the visible extent is then a multiple of 4
// except for a ragged N, handled by the scalar tail).
__global__ void __launch_bounds__(kRowThreads) row_stats_kernel(const float* __restrict__ scores, int64_t R,
                                                                 int64_t Np, int64_t N, int32_t pq, int32_t causal,
                                                                 float sl2, int32_t want_z, float* __restrict__ rmax,
                                                                 double* __restrict__ rz) {
    __shared__ float shf[32];
    __shared__ double shd[32];
    const bool vec = (N & 3) == 0;
    for (int64_t row = blockIdx.x; row < R; row += gridDim.x) {
        const int64_t vend = vis_end(row, Np, N, pq, causal);
        const int64_t v4 = vec ? vend / 4 : 0;
        const float* s = scores + row * N;
        const float4* s4 = reinterpret_cast<const float4*>(s);
        float m = -INFINITY;
        for (int64_t j = threadIdx.x; j < v4; j += kRowThreads) {
            const float4 x = __ldg(s4 + j);
            m = fmaxf(fmaxf(m, fmaxf(x.x, x.y)), fmaxf(x.z, x.w));
        }
        for (int64_t j = 4 * v4 + threadIdx.x; j < vend; j += kRowThreads) m = fmaxf(m, __ldg(s + j));
        m = block_max(m, shf);
        if (threadIdx.x == 0) rmax[row] = m;
        if (want_z) {
            double z = 0.0;
            for (int64_t j = threadIdx.x; j < v4; j += kRowThreads) {
                const float4 x = __ldg(s4 + j);
                z += (double)(exp2f((x.x - m) * sl2) + exp2f((x.y - m) * sl2)) +
                     (double)(exp2f((x.z - m) * sl2) + exp2f((x.w - m) * sl2));
            }
            for (int64_t j = 4 * v4 + threadIdx.x; j < vend; j += kRowThreads) z += (double)exp2f((__ldg(s + j) - m) * sl2);
            z = block_sum(z, shd);
            if (threadIdx.x == 0) rz[row] = z;
        }
    }
}

// minS filter (Eq. 3): bit j of row r set iff acc_rj >= max_r - alpha_raw (alpha/scale).
// A lane tests 4 consecutive keys (one 16-B load); 8 lanes OR their nibbles into a word.
__global__ void __launch_bounds__(kRowThreads) mins_filter_kernel(const float* __restrict__ scores, int64_t R,
                                                                   int64_t Np, int64_t N, int32_t pq, int32_t causal,
                                                                   const float* __restrict__ rmax, float alpha_raw,
                                                                   uint32_t* __restrict__ bitmask,
                                                                   int64_t words_per_row,
                                                                   unsigned long long* __restrict__ counts) {
    __shared__ double shd[32];
    const int lane = threadIdx.x & 31;
    const bool vec = (N & 3) == 0;
    for (int64_t row = blockIdx.x; row < R; row += gridDim.x) {
        const int64_t vend = vis_end(row, Np, N, pq, causal);
        const float thr = rmax[row] - alpha_raw;
        const float* s = scores + row * N;
        uint32_t* bm = bitmask + row * words_per_row;
        double cnt = 0.0;
        // words_per_row * 8 quads per row; every lane of the block walks the quads in order
        for (int64_t qd0 = 0; qd0 < words_per_row * 8; qd0 += kRowThreads) {
            const int64_t qd = qd0 + threadIdx.x;
            const int64_t j0 = 4 * qd;
            uint32_t nib = 0;
            if (j0 < vend) {
                if (vec && j0 + 4 <= vend) {
                    const float4 x = __ldg(reinterpret_cast<const float4*>(s + j0));
                    nib = (x.x >= thr ? 1u : 0u) | (x.y >= thr ? 2u : 0u) | (x.z >= thr ? 4u : 0u) | (x.w >= thr ? 8u : 0u);
                } else {
                    for (int b = 0; b < 4; ++b)
                        if (j0 + b < vend && __ldg(s + j0 + b) >= thr) nib |= 1u << b;
                }
            }
            uint32_t word = nib << (4 * (lane & 7));
            word |= __shfl_xor_sync(0xffffffffu, word, 1);
            word |= __shfl_xor_sync(0xffffffffu, word, 2);
            word |= __shfl_xor_sync(0xffffffffu, word, 4);
            if ((lane & 7) == 0 && qd / 8 < words_per_row) bm[qd / 8] = word;
            cnt += __popc(nib);
        }
        cnt = block_sum(cnt, shd);
        if (threadIdx.x == 0) counts[row] = (unsigned long long)cnt;
    }
}

// Values (key indices) and segment bounds for one batch of rows of the topP sort.
__global__ void topp_prepare_kernel(int64_t row0, int64_t nrows, int64_t Np, int64_t N, int32_t pq, int32_t causal,
                                    int32_t* __restrict__ vals, int64_t* __restrict__ seg_begin,
                                    int64_t* __restrict__ seg_end) {
    const int64_t total = nrows * N;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x)
        vals[x] = (int32_t)(x % N);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        seg_begin[r] = r * N;
        seg_end[r] = r * N + vis_end(row0 + r, Np, N, pq, causal);
    }
}

// topP cut on the sorted row: the smallest prefix whose cumulative mass reaches p*Z
// (zero-probability keys never taken); its keys' bits are set in the row bitmask.
__global__ void __launch_bounds__(kRowThreads) topp_cut_kernel(const float* __restrict__ skeys,
                                                                const int32_t* __restrict__ svals, int64_t row0,
                                                                int64_t nrows, int64_t Np, int64_t N, int32_t pq,
                                                                int32_t causal, float sl2, float top_p,
                                                                const float* __restrict__ rmax,
                                                                const double* __restrict__ rz,
                                                                uint32_t* __restrict__ bitmask, int64_t words_per_row,
                                                                unsigned long long* __restrict__ counts) {
    extern __shared__ uint32_t sbm[];  // [words_per_row] row bitmask
    __shared__ double wsum[kRowThreads / 32];
    __shared__ int64_t s_k;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t rr = blockIdx.x; rr < nrows; rr += gridDim.x) {
        const int64_t row = row0 + rr;
        const int64_t vend = vis_end(row, Np, N, pq, causal);
        const float m = rmax[row];
        const double target = (double)top_p * rz[row];
        const float* ks = skeys + rr * N;
        const int32_t* vs = svals + rr * N;
        for (int64_t x = threadIdx.x; x < words_per_row; x += kRowThreads) sbm[x] = 0u;
        if (threadIdx.x == 0) s_k = -1;
        __syncthreads();
        double run = 0.0;  // cumulative mass before the current block of kRowThreads keys
        int64_t k = vend;  // selected prefix length (all visible if p*Z is never reached)
        for (int64_t t0 = 0; t0 < vend; t0 += kRowThreads) {
            const int64_t t = t0 + threadIdx.x;
            const float e = t < vend ? exp2f((__ldg(ks + t) - m) * sl2) : 0.f;
            // block inclusive scan of e (fp64)
            double inc = e;
            for (int o = 1; o < 32; o <<= 1) {
                const double n = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += n;
            }
            if (lane == 31) wsum[w] = inc;
            __syncthreads();
            double pre = 0.0, tot = 0.0;
            for (int q = 0; q < kRowThreads / 32; ++q) {
                if (q < w) pre += wsum[q];
                tot += wsum[q];
            }
            const double cum = run + pre + inc;
            // first position reaching the target, or the first zero-probability key
            const bool hit = t < vend && (cum >= target || e == 0.f);
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            if (bal && lane == __ffs(bal) - 1) atomicMin((unsigned long long*)&s_k,
                                                         (unsigned long long)(e == 0.f ? t : t + 1));
            __syncthreads();
            if (s_k != -1) {
                k = s_k;
                break;
            }
            run += tot;
            __syncthreads();
        }
        __syncthreads();
        for (int64_t t = threadIdx.x; t < k; t += kRowThreads) {
            const int32_t j = __ldg(vs + t);
            atomicOr(&sbm[j >> 5], 1u << (j & 31));
        }
        __syncthreads();
        uint32_t* bm = bitmask + row * words_per_row;
        for (int64_t x = threadIdx.x; x < words_per_row; x += kRowThreads) bm[x] = sbm[x];
        if (threadIdx.x == 0) counts[row] = (unsigned long long)k;
        __syncthreads();
    }
}

int row_grid(int64_t rows) { return (int)std::min<int64_t>(rows, 148 * 8); }

}  // namespace

cudaError_t launch_naive_row_stats(const float* scores, int64_t R, int64_t Np, int64_t N, int32_t pq, int32_t causal,
                                   float sl2, int want_z, float* rmax, double* rz, cudaStream_t st) {
    if (R <= 0) return cudaSuccess;
    row_stats_kernel<<<row_grid(R), kRowThreads, 0, st>>>(scores, R, Np, N, pq, causal, sl2, want_z, rmax, rz);
    return cudaGetLastError();
}

cudaError_t launch_naive_mins(const float* scores, int64_t R, int64_t Np, int64_t N, int32_t pq, int32_t causal,
                              const float* rmax, float alpha_raw, uint32_t* bitmask, int64_t words_per_row,
                              unsigned long long* counts, cudaStream_t st) {
    if (R <= 0) return cudaSuccess;
    mins_filter_kernel<<<row_grid(R), kRowThreads, 0, st>>>(scores, R, Np, N, pq, causal, rmax, alpha_raw, bitmask,
                                                             words_per_row, counts);
    return cudaGetLastError();
}

int64_t naive_topp_batch_rows(int64_t R, int64_t N) {
    return std::max<int64_t>(1, std::min<int64_t>(R, (int64_t(1) << 29) / N));
}

size_t naive_topp_sort_temp_bytes(int64_t batch_rows, int64_t N) {
    size_t bytes = 0;
    const int64_t items = batch_rows * N;
    cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, bytes, (const float*)nullptr, (float*)nullptr,
                                                       (const int32_t*)nullptr, (int32_t*)nullptr, items,
                                                       batch_rows, (const int64_t*)nullptr, (const int64_t*)nullptr);
    return bytes;
}

cudaError_t launch_naive_topp(const float* scores, int64_t R, int64_t Np, int64_t N, int32_t pq, int32_t causal,
                              float sl2, float top_p, const float* rmax, const double* rz, float* skeys, int32_t* vals_in,
                              int32_t* vals_out, int64_t* seg_begin, int64_t* seg_end, void* temp, size_t temp_bytes,
                              uint32_t* bitmask, int64_t words_per_row, unsigned long long* counts, cudaStream_t st) {
    const int64_t B = naive_topp_batch_rows(R, N);
    const int smem = (int)(words_per_row * 4);
    cudaError_t e = cudaFuncSetAttribute(topp_cut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    for (int64_t r0 = 0; r0 < R; r0 += B) {
        const int64_t nb = std::min<int64_t>(B, R - r0);
        topp_prepare_kernel<<<1184, 256, 0, st>>>(r0, nb, Np, N, pq, causal, vals_in, seg_begin, seg_end);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        size_t tb = temp_bytes;
        e = cub::DeviceSegmentedRadixSort::SortPairsDescending(temp, tb, scores + r0 * N, skeys, vals_in, vals_out,
                                                               nb * N, nb, seg_begin, seg_end, 0, 32, st);
        if (e != cudaSuccess) return e;
        topp_cut_kernel<<<row_grid(nb), kRowThreads, smem, st>>>(skeys, vals_out, r0, nb, Np, N, pq, causal, sl2,
                                                                  top_p, rmax, rz, bitmask, words_per_row, counts);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace va
