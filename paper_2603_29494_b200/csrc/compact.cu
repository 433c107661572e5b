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

#include <algorithm>

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

template <int kEmitWarps, bool STREAM>
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
        auto ld = [&](const uint32_t* a) { return STREAM ? __ldcs(a) : __ldg(a); };
        uint32_t next = lane < nwords ? ld(src + lane) : 0u;  // software-pipelined by one round
        for (int64_t w0 = 0; w0 < nwords; w0 += 32) {
            uint32_t word = next;
            next = (w0 + 32 + lane < nwords) ? ld(src + w0 + 32 + lane) : 0u;
            const int pc = __popc(word);
            int incl = pc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int n = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += n;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            int pos = incl;  // bits are taken from the top: fill [incl - pc, incl) backwards
            const int32_t kbase = (int32_t)((w0 + lane) * 32);
            while (word) {
                const int bit = 31 - __clz(word);
                stage[w][--pos] = kbase + bit;
                word ^= 1u << bit;
            }
            __syncwarp();
            for (int t = lane; t < total; t += 32) {
                if constexpr (STREAM) __stcs(indices + out + t, stage[w][t]);
                else indices[out + t] = stage[w][t];
            }
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
    emit_kernel<kEmitWarps, false><<<(unsigned)blocks, kEmitWarps * 32, 0, st>>>(
        bitmask, words_per_row, offsets, d_nnz, cap, indices, BH, Np, N, pq, causal);
    return cudaGetLastError();
}

// Emission beside the attention kernel (vecattn_forward): one 2-warp CTA per SM, 8 KB of
// shared memory, so it fits next to the persistent attention CTA and runs on that SM's
// spare issue slots; bitmask reads and index stores are streamed (evict-first) so they do
// not displace the K/V rows the attention gathers from L2.
cudaError_t launch_emit_shadow(const uint32_t* bitmask, int64_t words_per_row, const int64_t* offsets,
                               const int64_t* d_nnz, int64_t cap, int32_t* indices, int64_t BH, int64_t Np,
                               int64_t N, int32_t pq, int32_t causal, int sms, cudaStream_t st) {
    emit_kernel<2, true><<<(unsigned)std::max(1, sms), 64, 0, st>>>(bitmask, words_per_row, offsets, d_nnz, cap,
                                                                    indices, BH, Np, N, pq, causal);
    return cudaGetLastError();
}

// ------------------------------------------------------------------- fused plan
// One CTA per 256-row attention item (G = 256/P_q selection rows).  From the
// selection bitmask it emits the attention worklist of the item (attn.cu): the sorted
// union of its rows' selections with one membership bit per row (entry = key |
// bits << 28), split into three segments -- keys used by both 128-row tiles, by tile 0
// only, by tile 1 only -- at the item's CSR base; segment lengths -> wl_len[3*item +
// {0,1,2}] (if nnz <= wl_cap).  (CSR indices come from emit_kernel.)
// Rounds of 256 bitmask words (lane = word, coalesced loads); per round a block-wide
// exclusive scan of the 3 segment counts, entries staged in shared memory, then
// written out coalesced.
constexpr int kPlanThreads = 256;

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(const uint32_t* __restrict__ bitmask,
                                                            int64_t words_per_row,
                                                            const int64_t* __restrict__ offsets,
                                                            const int64_t* __restrict__ d_nnz, int64_t wl_cap,
                                                            uint32_t* __restrict__ wl, int32_t* __restrict__ wl_len,
                                                            int64_t Np, int64_t n_it, int64_t N, int32_t pq,
                                                            int32_t causal) {
    __shared__ int sh[3][kPlanThreads / 32];
    __shared__ uint32_t stage[kPlanThreads * 32];  // worst case: every bit of a round in one segment
    const int64_t item = blockIdx.x;
    const int64_t bh = item / n_it, it = item % n_it;
    const int G = 256 / pq;
    const int64_t i0 = it * G;
    const int nb = (int)min((int64_t)G, Np - i0);
    const int64_t r0 = bh * Np + i0;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (*d_nnz > wl_cap) {
        if (tid == 0) wl_len[3 * item] = wl_len[3 * item + 1] = wl_len[3 * item + 2] = 0;
        return;
    }
    int64_t vwords[4];
    int64_t wmax = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const int64_t i = i0 + b;
        const int64_t vis = b < nb ? (causal ? min(N, (i + 1) * (int64_t)pq) : N) : 0;
        vwords[b] = (vis + 31) / 32;
        wmax = max(wmax, vwords[b]);
    }
    const bool quad = G == 4;
    // pass 1: segment totals (needed to place segments 1 and 2)
    int c3[3] = {0, 0, 0};
    for (int64_t x = tid; x < wmax; x += kPlanThreads) {
        uint32_t bw[4];
#pragma unroll
        for (int b = 0; b < 4; ++b)
            bw[b] = (b < nb && x < vwords[b]) ? __ldg(bitmask + (r0 + b) * words_per_row + x) : 0u;
        const uint32_t u0 = quad ? (bw[0] | bw[1]) : bw[0];
        const uint32_t u1 = quad ? (bw[2] | bw[3]) : bw[1];
        c3[0] += __popc(u0 & u1);
        c3[1] += __popc(u0 & ~u1);
        c3[2] += __popc(u1 & ~u0);
    }
    int tot[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        int v = c3[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) sh[k][w] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        int t = 0;
        for (int x = 0; x < kPlanThreads / 32; ++x) t += sh[k][x];
        tot[k] = t;
    }
    __syncthreads();
    const int64_t base = offsets[r0];
    int64_t run[3] = {base, base + tot[0], base + tot[0] + tot[1]};
    // pass 2: rounds of kPlanThreads words.  The three segment counts of a word are packed in
    // one 64-bit value (21 bits each; a round holds at most 8192 keys), so a single block scan
    // places all three; the round's entries are staged segment after segment (the segments
    // are disjoint, so at most 8192 entries) and written out coalesced.
    __shared__ unsigned long long sh64[kPlanThreads / 32];
    uint32_t nx[4];  // next round's words (software-pipelined by one round)
#pragma unroll
    for (int b = 0; b < 4; ++b) nx[b] = (b < nb && tid < vwords[b]) ? __ldg(bitmask + (r0 + b) * words_per_row + tid) : 0u;
    for (int64_t x0 = 0; x0 < wmax; x0 += kPlanThreads) {
        const int64_t x = x0 + tid;
        uint32_t bw[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            bw[b] = nx[b];
            const int64_t xn = x + kPlanThreads;
            nx[b] = (b < nb && xn < vwords[b]) ? __ldg(bitmask + (r0 + b) * words_per_row + xn) : 0u;
        }
        const uint32_t u0 = quad ? (bw[0] | bw[1]) : bw[0];
        const uint32_t u1 = quad ? (bw[2] | bw[3]) : bw[1];
        const uint32_t seg[3] = {u0 & u1, u0 & ~u1, u1 & ~u0};
        const unsigned long long cnt = (unsigned long long)__popc(seg[0]) |
                                       ((unsigned long long)__popc(seg[1]) << 21) |
                                       ((unsigned long long)__popc(seg[2]) << 42);
        unsigned long long incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long n = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += n;
        }
        if (lane == 31) sh64[w] = incl;
        __syncthreads();
        unsigned long long before = 0, rtot = 0;
#pragma unroll
        for (int y = 0; y < kPlanThreads / 32; ++y) {
            const unsigned long long t = sh64[y];
            before += (y < w) ? t : 0ull;
            rtot += t;
        }
        const unsigned long long excl = before + incl - cnt;
        constexpr unsigned long long F = (1ull << 21) - 1ull;
        const int rt0 = (int)(rtot & F), rt1 = (int)((rtot >> 21) & F), rt2 = (int)(rtot >> 42);
        const int soff[3] = {0, rt0, rt0 + rt1};
        const uint32_t kbase = (uint32_t)(x * 32);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            // bits taken from the top, written backwards into [start, start + popc)
            int pos = soff[k] + (int)(((excl + cnt) >> (21 * k)) & F);
            uint32_t m = seg[k];
            while (m) {
                const int bit = 31 - __clz(m);
                const uint32_t mem = ((bw[0] >> bit) & 1u) | (((bw[1] >> bit) & 1u) << 1) |
                                     (((bw[2] >> bit) & 1u) << 2) | (((bw[3] >> bit) & 1u) << 3);
                stage[--pos] = (kbase + (uint32_t)bit) | (mem << 28);
                m ^= 1u << bit;
            }
        }
        __syncthreads();
        // one coalesced copy loop per segment (pointer-stepped: fewer instructions per entry than
        // one loop that picks the segment of every entry)
        {
            uint32_t* d0 = wl + run[0];
            for (int t = tid; t < rt0; t += kPlanThreads) d0[t] = stage[t];
            uint32_t* d1 = wl + run[1];
            const uint32_t* s1 = stage + rt0;
            for (int t = tid; t < rt1; t += kPlanThreads) d1[t] = s1[t];
            uint32_t* d2 = wl + run[2];
            const uint32_t* s2 = stage + rt0 + rt1;
            for (int t = tid; t < rt2; t += kPlanThreads) d2[t] = s2[t];
        }
        run[0] += rt0;
        run[1] += rt1;
        run[2] += rt2;
        __syncthreads();
    }
    if (tid == 0) {
        wl_len[3 * item] = tot[0];
        wl_len[3 * item + 1] = tot[1];
        wl_len[3 * item + 2] = tot[2];
    }
}

// ------------------------------------------------------------------- item order
// One CTA per head: the head's items inside the window [lo, hi) of the flattened items, sorted
// in shared memory (bitonic) by (weight descending, item ascending) -- weight = tile-chunks
// 2 * chunks(both tiles) + chunks(tile 0) + chunks(tile 1) of 64 keys, or (by_position, the
// causal default: later items see more keys) the item's position -- and written at the head's
// offset in the window: order[pos] = bh * n_mt + it.
constexpr int kLptThreads = 1024;
__global__ void __launch_bounds__(kLptThreads) lpt_order_kernel(const int32_t* __restrict__ wl_len, int64_t n_mt,
                                                                int64_t lo, int64_t hi, int32_t by_position,
                                                                int32_t* __restrict__ order) {
    __shared__ unsigned long long key[kLptMaxItems];
    const int64_t bh = blockIdx.x;
    const int64_t h0 = bh * n_mt;
    const int64_t a = max(lo, h0) - h0, b = min(hi, h0 + n_mt) - h0;  // items [a, b) of this head
    if (b <= a) return;
    const int64_t n = b - a;
    int32_t* out = order + (max(lo, h0) - lo);
    if (n_mt > kLptMaxItems) {  // position order, reversed (longest first when causal)
        for (int64_t i = threadIdx.x; i < n; i += kLptThreads) out[i] = (int32_t)(h0 + b - 1 - i);
        return;
    }
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int i = threadIdx.x; i < n2; i += kLptThreads) {
        unsigned long long k = ~0ull;  // padding sorts last
        if (i < n) {
            const int64_t it = a + i;
            uint32_t w;
            if (by_position) {
                w = (uint32_t)it;
            } else {
                const int32_t* l = wl_len + 3 * (h0 + it);
                w = 2u * (uint32_t)((l[0] + 63) / 64) + (uint32_t)((l[1] + 63) / 64) + (uint32_t)((l[2] + 63) / 64);
            }
            k = ((unsigned long long)(0xFFFFFFFFu - w) << 32) | (uint32_t)it;
        }
        key[i] = k;
    }
    __syncthreads();
    for (int size = 2; size <= n2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < n2; i += kLptThreads) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const unsigned long long x = key[i], y = key[j];
                    if ((x > y) == up) {
                        key[i] = y;
                        key[j] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += kLptThreads) out[i] = (int32_t)(h0 + (int64_t)(key[i] & 0xFFFFFFFFull));
}

cudaError_t launch_lpt_order(const int32_t* wl_len, int64_t BH, int64_t n_mt, int64_t lo, int64_t hi,
                             int32_t by_position, int32_t* order, cudaStream_t st) {
    if (BH <= 0 || n_mt <= 0 || hi <= lo) return cudaSuccess;
    lpt_order_kernel<<<(unsigned)BH, kLptThreads, 0, st>>>(wl_len, n_mt, lo, hi, by_position, order);
    return cudaGetLastError();
}

cudaError_t launch_plan(const uint32_t* bitmask, int64_t words_per_row, const int64_t* offsets, const int64_t* d_nnz,
                        int64_t wl_cap, uint32_t* wl, int32_t* wl_len, int64_t BH, int64_t Np, int64_t N, int32_t pq,
                        int32_t causal, cudaStream_t st) {
    const int64_t n_it = (N + 255) / 256;
    const int64_t items = BH * n_it;
    if (items <= 0) return cudaSuccess;
    plan_kernel<<<(unsigned)items, kPlanThreads, 0, st>>>(bitmask, words_per_row, offsets, d_nnz, wl_cap, wl, wl_len,
                                                          Np, n_it, N, pq, causal);
    return cudaGetLastError();
}

}  // namespace va
