// compact.cu — index emission: per-block selection bitmask -> CSR (I, C of Alg. 1).
//
// PAPER.md P:673-676 / Alg. 1: per query block the kernel emits the
// important-vector index set Idx(i) and its count C_i.  Stored as CSR (reading
// R9: ascending, unique): offsets int64 [R+1] (exclusive scan of the counts
// produced by select.cu's epilogue) and indices int32 [nnz].
// HBM-bound: reads the bitmask rows up to each row's visible extent, writes 4 B
// per selected (block, key) pair (the Theta(N^2 (1-rho)/P_q) term of P:277).
#include "common.cuh"
#include "kernels.cuh"

namespace va {

// Single-CTA exclusive scan over R row counts (R = B*Hq*N_p, <= a few 1e5).
__global__ void __launch_bounds__(1024) scan_kernel(const unsigned long long* __restrict__ counts, int64_t R,
                                                    int64_t* __restrict__ offsets, int64_t* __restrict__ d_nnz) {
    __shared__ unsigned long long warp_tot[32];
    const int t = threadIdx.x;
    const int64_t per = (R + 1023) / 1024;
    const int64_t lo = min(R, t * per), hi = min(R, lo + per);
    unsigned long long s = 0;
    for (int64_t r = lo; r < hi; ++r) s += counts[r];
    // block exclusive scan of s
    const int lane = t & 31, w = t >> 5;
    unsigned long long inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long n = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += n;
    }
    if (lane == 31) warp_tot[w] = inc;
    __syncthreads();
    if (w == 0) {
        unsigned long long v = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long n = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += n;
        }
        warp_tot[lane] = v;  // inclusive over warps
    }
    __syncthreads();
    unsigned long long run = (inc - s) + (w ? warp_tot[w - 1] : 0ull);
    if (t == 0) offsets[0] = 0;
    for (int64_t r = lo; r < hi; ++r) {
        run += counts[r];
        offsets[r + 1] = (int64_t)run;
    }
    if (t == 1023) *d_nnz = (int64_t)warp_tot[31];
}

// One warp per row; 32 bitmask words (1024 keys) per round, staged in shared memory
// so the index stores are coalesced.
constexpr int kEmitWarps = 8;

__global__ void __launch_bounds__(kEmitWarps * 32) emit_kernel(const uint32_t* __restrict__ bitmask,
                                                                 int64_t words_per_row,
                                                                 const int64_t* __restrict__ offsets,
                                                                 const int64_t* __restrict__ d_nnz, int64_t cap,
                                                                 int32_t* __restrict__ indices, int64_t BH,
                                                                 int64_t Np, int64_t N, int32_t pq,
                                                                 int32_t causal) {
    __shared__ int32_t stage[kEmitWarps][1024];
    if (*d_nnz > cap) return;  // capacity protocol: caller re-allocates and calls again
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t R = BH * Np;
    for (int64_t row = (int64_t)blockIdx.x * kEmitWarps + w; row < R; row += (int64_t)gridDim.x * kEmitWarps) {
        const int64_t i = row % Np;
        const int64_t vis = causal ? min(N, (i + 1) * (int64_t)pq) : N;
        const int64_t nwords = (vis + 31) / 32;
        const uint32_t* src = bitmask + row * words_per_row;
        int64_t out = offsets[row];
        for (int64_t w0 = 0; w0 < nwords; w0 += 32) {
            uint32_t word = (w0 + lane < nwords) ? __ldg(src + w0 + lane) : 0u;
            const int pc = __popc(word);
            int incl = pc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int n = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += n;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            int pos = incl - pc;
            const int32_t kbase = (int32_t)((w0 + lane) * 32);
            while (word) {
                const int bit = __ffs(word) - 1;
                stage[w][pos++] = kbase + bit;
                word &= word - 1;
            }
            __syncwarp();
            for (int t = lane; t < total; t += 32) indices[out + t] = stage[w][t];
            __syncwarp();
            out += total;
        }
    }
}

cudaError_t launch_scan(const unsigned long long* counts, int64_t R, int64_t* offsets, int64_t* d_nnz,
                        cudaStream_t st) {
    scan_kernel<<<1, 1024, 0, st>>>(counts, R, offsets, d_nnz);
    return cudaGetLastError();
}

cudaError_t launch_emit(const uint32_t* bitmask, int64_t words_per_row, const int64_t* offsets,
                        const int64_t* d_nnz, int64_t cap, int32_t* indices, int64_t BH, int64_t Np, int64_t N,
                        int32_t pq, int32_t causal, cudaStream_t st) {
    const int64_t R = BH * Np;
    int64_t blocks = (R + kEmitWarps - 1) / kEmitWarps;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    emit_kernel<<<(unsigned)blocks, kEmitWarps * 32, 0, st>>>(bitmask, words_per_row, offsets, d_nnz, cap, indices,
                                                              BH, Np, N, pq, causal);
    return cudaGetLastError();
}

}  // namespace va
