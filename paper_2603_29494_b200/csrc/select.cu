// select.cu — important-vector selection ("TilingSelect" + minS / topK), sm_100a.
//
// The pooled-score GEMM S = Q_p K^T (Alg. 1) runs on
// tcgen05 tensor cores with the 128 x BN score tile held in TMEM; the filter is
// applied in the epilogue straight out of TMEM, so the estimated attention map is
// never written to HBM (Sec. 3.1.3).  Only a 1-bit-per-key selection
// mask leaves the chip; compact.cu turns it into sorted index lists (I, C of
// Alg. 1).
//
// CTA = one work unit (head bh, 128 pooled rows, key segment).  Warp roles:
//   warp 0  TMA producer: Q_p tile once, then K tiles [BN x D] into a STAGES ring
//   warp 1  TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 2-5 epilogue: thread = pooled row (TMEM lane), 2 TMEM accumulators so the
//           epilogue of tile t overlaps the MMA of tile t+1.
// Epilogues (template EPI):
//   EPI_ALG1   Alg. 1: running row max per B_K chunk, reset every G_K
//              tiles (reading R2), keep s >= m - alpha AFTER the update
//              (readings R1 '>=' and R3).
//   EPI_MAX / EPI_THRESH   Eq. 3: global row max, then fixed threshold.
//   EPI_TOPK_HIST / EPI_TOPK_EMIT   topK: 4 radix passes over
//              order-preserving fp32 keys, then emit with ties -> lowest index (R12).
//   EPI_SCORES debug dump of the raw accumulators (tests only).
// Comparisons use raw accumulators: s = scale*acc with scale > 0, so
// s >= m - alpha  <=>  acc >= m_acc - alpha/scale (alpha_raw, computed on host).
// Causal (reading R5): keys j > L_i = min(N,(i+1)P_q)-1 are excluded before max
// and filter; keys >= N (ragged tail, R7) likewise.
#include "common.cuh"
#include "kernels.cuh"

#include <math.h>
#include <stdlib.h>

namespace va {

namespace {

// w0 TMA producer, w1 MMA issuer, then the epilogue warps: 4 (thread = pooled row), or 8 for
// the TOPK histogram passes, whose two warp sets take alternate 64-key chunks of every tile
// and update the same per-row histogram with shared-memory atomics.
template <int EPI>
constexpr int epi_warps() { return (EPI == EPI_TOPK_HIST || EPI == EPI_TK_SHIST || EPI == EPI_TK_CAND) ? 8 : 4; }
template <int EPI>
constexpr int sel_threads() { return 64 + 32 * epi_warps<EPI>(); }

template <int D, int BN, int STAGES, int EPI>
struct SelCfg {
    static constexpr int kCB = D / 64;                       // 128-byte column blocks
    static constexpr int kQBytes = kCB * 128 * 128;          // Q_p tile
    static constexpr int kKStageBytes = kCB * BN * 128;      // one K tile
    static constexpr int kHistBytes = (EPI == EPI_TOPK_HIST || EPI == EPI_TK_SHIST) ? 256 * 128 * 4
                                      : (EPI == EPI_TK_CAND ? 2 * 64 * 128 * 4 : 0);  // CAND: score staging per warp set
    static constexpr int kOffQ = 0;
    static constexpr int kOffK = kQBytes;
    static constexpr int kOffHist = kOffK + STAGES * kKStageBytes;
    static constexpr int kOffBar = kOffHist + kHistBytes;
    static constexpr int kNumBars = 1 + 2 * STAGES + 4;
    static constexpr int kSmem = kOffBar + kNumBars * 8 + 16;
    static constexpr uint32_t kTmemCols = 2 * BN;
    static constexpr uint32_t kIdesc = make_idesc_bf16(128, BN, 0, 0);
};

VA_DEV float fmax3(float a, float b, float c) { return fmaxf(fmaxf(a, b), c); }

}  // namespace

template <int D, int BN, int STAGES, int EPI, int BK>
__global__ void __launch_bounds__(sel_threads<EPI>(), 1) select_kernel(const __grid_constant__ SelectParams p) {
    using C = SelCfg<D, BN, STAGES, EPI>;
    extern __shared__ __align__(1024) uint8_t smem[];

    // ---- unit decode: unit = ((bh * n_mt) + mt) * n_seg + seg
    const int64_t unit = blockIdx.x;
    const int64_t seg = unit % p.n_seg;
    const int64_t mt = (unit / p.n_seg) % p.n_mt;
    const int64_t bh = unit / (p.n_seg * p.n_mt);
    const int64_t m0 = mt * 128;
    const int64_t row_hi = min(p.Np, m0 + 128);  // exclusive
    // sampled TOPK passes: key j of this pass is real key j * stride (R5 visibility on real keys)
    const int64_t stride = p.key_stride > 1 ? p.key_stride : 1;
    const int64_t kend_tile = p.causal ? min(p.N, (min(p.N_real, row_hi * (int64_t)p.pq) + stride - 1) / stride) : p.N;
    const int64_t k_begin = seg * p.seg_len;
    const int64_t k_end = min(k_begin + p.seg_len, kend_tile);
    if (k_begin >= k_end) return;  // uniform: causal units above the diagonal
    const int n_tiles = (int)((k_end - k_begin + BN - 1) / BN);
    const int64_t b = bh / p.Hq;
    const int64_t h = bh % p.Hq;
    const int64_t bh_kv = b * p.Hkv + h / (p.Hq / p.Hkv);
    if constexpr (EPI == EPI_TOPK_HIST || EPI == EPI_TOPK_EMIT) {
        // fallback of the windowed TOPK: only tiles with a row whose window missed
        if (p.only_failed) {
            if (*p.tk_nfail == 0) return;
            const int64_t rr = m0 + threadIdx.x;
            const int f = (threadIdx.x < 128 && rr < row_hi) ? (int)p.tk_fail[bh * p.Np + rr] : 0;
            if (!__syncthreads_or(f)) return;
        }
    }

    uint8_t* sQ = smem + C::kOffQ;
    uint8_t* sK = smem + C::kOffK;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* q_full = bars;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = bars + 1 + STAGES;
    uint64_t* acc_full = bars + 1 + 2 * STAGES;
    uint64_t* acc_empty = bars + 3 + 2 * STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();

    if (threadIdx.x == 0) {
        if ((smem_u32(smem) & 1023u) != 0) __trap();  // SW128 tiles need 1024-B alignment
        mbar_init(q_full, 1);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&acc_full[s], 1);
            mbar_init(&acc_empty[s], 32 * epi_warps<EPI>());
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ================================================================ producer
        if (elect_one()) {
            tma_prefetch_desc(&p.tm_qp);
            tma_prefetch_desc(&p.tm_k);
            mbar_arrive_expect_tx(q_full, C::kQBytes);
#pragma unroll
            for (int cb = 0; cb < C::kCB; ++cb)
                tma_load_3d(sQ + cb * 128 * 128, &p.tm_qp, q_full, cb * 64, (int)m0, (int)bh);
            for (int t = 0; t < n_tiles; ++t) {
                const int s = t % STAGES;
                if (t >= STAGES) mbar_wait(&k_empty[s], ((t / STAGES) - 1) & 1);
                mbar_arrive_expect_tx(&k_full[s], C::kKStageBytes);
                const int key0 = (int)(k_begin + (int64_t)t * BN);
#pragma unroll
                for (int cb = 0; cb < C::kCB; ++cb)
                    tma_load_3d(sK + s * C::kKStageBytes + cb * BN * 128, &p.tm_k, &k_full[s], cb * 64, key0,
                                (int)bh_kv);
            }
        }
    } else if (warp == 1) {
        // ================================================================ MMA issuer
        if (elect_one()) {
            mbar_wait(q_full, 0);
            tc_fence_after();
            const uint32_t qa = smem_u32(sQ);
            for (int t = 0; t < n_tiles; ++t) {
                const int s = t % STAGES;
                const int buf = t & 1;
                mbar_wait(&k_full[s], (t / STAGES) & 1);
                if (t >= 2) mbar_wait(&acc_empty[buf], ((t >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t ka = smem_u32(sK + s * C::kKStageBytes);
                const uint32_t d_tmem = tmem_base + (uint32_t)(buf * BN);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint64_t adesc = make_sdesc(qa + (kk >> 2) * 128 * 128 + (kk & 3) * 32, 16, 1024);
                    const uint64_t bdesc = make_sdesc(ka + (kk >> 2) * BN * 128 + (kk & 3) * 32, 16, 1024);
                    mma_bf16_ss(d_tmem, adesc, bdesc, C::kIdesc, kk > 0 ? 1u : 0u);
                }
                mma_commit(&k_empty[s]);
                mma_commit(&acc_full[buf]);
            }
        }
        __syncwarp();
    } else {
        // ================================================================ epilogue
        const uint32_t quad = warp & 3u;
        const int eset = ((int)warp - 2) >> 2;     // epilogue warp set (TOPK_HIST: 2 sets)
        const int r = (int)(quad * 32 + lane);
        const int64_t i = m0 + r;                  // pooled row within head
        const int64_t grow = bh * p.Np + i;        // global row id
        const bool row_ok = i < p.Np && !((EPI == EPI_TOPK_HIST || EPI == EPI_TOPK_EMIT) && p.only_failed &&
                                          p.tk_fail[grow] == 0u);
        const int64_t vis_real = p.causal ? min(p.N_real, (i + 1) * (int64_t)p.pq) : p.N_real;
        const int64_t vis_end = (vis_real + stride - 1) / stride;  // visible keys of this pass
        const float alpha_raw = p.alpha_raw[h];
        const int64_t G = (int64_t)p.bk * (int64_t)p.gk;
        int64_t next_reset = k_begin;              // Alg. 1 group boundaries (multiples of G)
        float m_run = -INFINITY;                   // ALG1 running max / EPI_MAX row max
        float span_mx = -INFINITY;                 // ALG1, B_K > 64: rowmax of the current sub-tile
        if (EPI == EPI_ALG1 && p.split && row_ok) {
            // K-split of a single-group row (G >= N): this segment continues the group that
            // started at key 0, so the running max starts at the max of the earlier segments
            // (Alg. 1's m_S is the max over every earlier visible key of the group).
            for (int64_t s2 = 0; s2 < seg; ++s2)
                m_run = fmaxf(m_run, f32_from_order_key(p.segmax[grow * p.n_seg + s2]));
            next_reset = (k_begin + G - 1) / G * G;
        }
        float thr_fixed = 0.f;
        float mn_run = INFINITY;                   // EPI_TK_MINMAX row min
        float tk_a = 0.f, tk_b = 0.f;              // SHIST: top*invw, invw; CAND: lo, hi
        uint32_t above = 0, ncand = 0;             // CAND counters
        float cb_v[4] = {0.f, 0.f, 0.f, 0.f};      // CAND: buffered candidates (scores, indices)
        int32_t cb_i[4] = {0, 0, 0, 0};
        uint32_t nb = 0;
        if constexpr (EPI == EPI_TK_SHIST) {
            if (row_ok) {
                tk_b = p.tk_invw[grow];
                tk_a = p.tk_top[grow] * tk_b;
            }
            if (eset == 0)
                for (int bin = 0; bin < 256; ++bin) reinterpret_cast<uint32_t*>(smem + C::kOffHist)[bin * 128 + r] = 0u;
            named_bar_sync(1, 32 * epi_warps<EPI>());  // zeroed before either warp set updates it
        }
        if constexpr (EPI == EPI_TK_CAND) {
            if (row_ok) {
                tk_a = p.tk_lo[grow];
                tk_b = p.tk_hi[grow];
            }
        }
        // CAND: this (row, key segment)'s candidate slice; subcap = cand_cap / n_seg
        // (two warp sets: slice (seg, set) of cand_cap / (2 n_seg) entries per row)
        const int64_t subcap = (EPI == EPI_TK_CAND) ? p.cand_cap / (2 * p.n_seg) : 0;
        const int64_t slice = 2 * seg + eset;
        float* cand_row = (EPI == EPI_TK_CAND) ? p.tk_cand + grow * p.cand_cap + slice * subcap : nullptr;
        int32_t* cidx_row = (EPI == EPI_TK_CAND) ? p.tk_cidx + grow * p.cand_cap + slice * subcap : nullptr;
        const bool vec_ok = (EPI == EPI_TK_CAND) && (subcap & 3) == 0 && ((uintptr_t)cand_row & 15u) == 0 &&
                            ((uintptr_t)cidx_row & 15u) == 0;
        uint32_t tk_prefix = 0, tk_krem = 0, tk_taken = 0;
        unsigned long long cnt = 0;
        uint32_t* hist = reinterpret_cast<uint32_t*>(smem + C::kOffHist);

        if constexpr (EPI == EPI_THRESH) {
            if (row_ok) thr_fixed = f32_from_order_key(p.rowmax[grow]) - alpha_raw;
        }
        if constexpr (EPI == EPI_TOPK_HIST || EPI == EPI_TOPK_EMIT) {
            if (row_ok) {
                if (EPI == EPI_TOPK_HIST && p.pass == 0) {
                    int64_t ki;
                    if (p.topk > 0) ki = min(p.topk, vis_real);
                    else {
                        ki = (int64_t)floor((double)p.keep_frac * (double)vis_real + 0.5);
                        ki = max((int64_t)1, min(ki, vis_real));
                    }
                    tk_prefix = 0;
                    tk_krem = (uint32_t)ki;
                } else {
                    tk_prefix = p.tk_prefix[grow];
                    tk_krem = p.tk_krem[grow];
                }
            }
            if constexpr (EPI == EPI_TOPK_HIST) {
                if (eset == 0)
                    for (int bin = 0; bin < 256; ++bin) hist[bin * 128 + r] = 0u;  // own column only
                named_bar_sync(1, 32 * epi_warps<EPI>());                       // zeroed before any update
            }
        }

        for (int t = 0; t < n_tiles; ++t) {
            const int buf = t & 1;
            mbar_wait(&acc_full[buf], (t >> 1) & 1);
            tc_fence_after();
            const int64_t key0 = k_begin + (int64_t)t * BN;
            uint32_t words[BN / 32];
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) {
                if constexpr (epi_warps<EPI>() == 8) {
                    if ((c & 1) != eset) continue;  // the other warp set's 64-key chunk
                }
                uint32_t va_[32], vb_[32];
                const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + (uint32_t)(buf * BN + c * 64);
                tmem_ld32(taddr, va_);
                tmem_ld32(taddr + 32, vb_);
                tmem_ld_wait();
                float v[64];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    v[j] = __uint_as_float(va_[j]);
                    v[32 + j] = __uint_as_float(vb_[j]);
                }
                const int64_t kc = key0 + c * 64;                 // first key of this 64-chunk
                const int64_t nv64 = vis_end - kc;                // visible prefix length
                const int nvis = row_ok ? (int)max((int64_t)0, min((int64_t)64, nv64)) : 0;
                uint32_t w0 = 0, w1 = 0;

                if constexpr (EPI == EPI_SCORES) {
                    if (row_ok) {
                        float* dst = p.scores_out + grow * p.N + kc;
                        if ((p.N & 3) == 0 && kc + 64 <= p.N) {  // 16-B stores (row-contiguous)
#pragma unroll
                            for (int j = 0; j < 64; j += 4)
                                *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 64; ++j)
                                if (kc + j < p.N) dst[j] = v[j];
                        }
                    }
                } else if constexpr (EPI == EPI_ALG1) {
                    if (nvis < 64) {
#pragma unroll
                        for (int j = 0; j < 64; ++j)
                            if (j >= nvis) v[j] = -INFINITY;
                    }
                    // rowmax of every B_K sub-tile first (independent chains), then Alg. 1's
                    // sequential running max and threshold per sub-tile.  B_K > 64: the sub-tile
                    // spans BK / 64 chunks of this TMEM tile (BK divides BN), so its rowmax is
                    // taken once, at its first chunk, by reading the later chunks ahead.
                    constexpr int kSub = BK < 64 ? BK : 64;
                    float gmx[64 / kSub];
                    if constexpr (BK > 64) {
                        if ((c * 64) % BK == 0) {
                            float a = -INFINITY, b = -INFINITY;
#pragma unroll
                            for (int j = 0; j < 64; j += 4) {
                                a = fmax3(a, v[j], v[j + 1]);
                                b = fmax3(b, v[j + 2], v[j + 3]);
                            }
#pragma unroll 1
                            for (int c2 = 1; c2 < BK / 64; ++c2) {
                                uint32_t ua[32], ub[32];
                                tmem_ld32(taddr + c2 * 64, ua);
                                tmem_ld32(taddr + c2 * 64 + 32, ub);
                                tmem_ld_wait();
                                const int64_t nv2 = vis_end - (kc + c2 * 64);
                                const int n2 = row_ok ? (int)max((int64_t)0, min((int64_t)64, nv2)) : 0;
#pragma unroll
                                for (int j = 0; j < 32; ++j) {
                                    if (j < n2) a = fmaxf(a, __uint_as_float(ua[j]));
                                    if (32 + j < n2) b = fmaxf(b, __uint_as_float(ub[j]));
                                }
                            }
                            span_mx = fmaxf(a, b);
                        }
                        gmx[0] = span_mx;
                    } else {
#pragma unroll
                        for (int g = 0; g < 64 / BK; ++g) {
                            float a = -INFINITY, b = -INFINITY;
#pragma unroll
                            for (int j = 0; j < BK; j += 4) {
                                a = fmax3(a, v[g * BK + j], v[g * BK + j + 1]);
                                b = fmax3(b, v[g * BK + j + 2], v[g * BK + j + 3]);
                            }
                            gmx[g] = fmaxf(a, b);
                        }
                    }
                    // keep = s >= m_S - alpha (R1) <=> the sign bit of s - thr is clear:
                    // for finite thr the IEEE difference is negative exactly when s < thr (no
                    // underflow to -0 with gradual underflow; s = -inf gives -inf).  The sign
                    // bits are shifted in (funnel shift) and inverted/bit-reversed per word.
                    uint32_t sg0 = 0u, sg1 = 0u;
#pragma unroll
                    for (int sub = 0; sub < 64; sub += kSub) {
                        if (kc + sub == next_reset) {  // new group of G_K tiles: m_S <- -inf
                            m_run = -INFINITY;
                            next_reset += G;
                        }
                        m_run = fmaxf(m_run, gmx[sub / kSub]);    // m_S <- max(m_S, rowmax(S_tile))
                        const float nthr = alpha_raw - m_run;     // -(m_S - alpha)
#pragma unroll
                        for (int j = sub; j < sub + kSub; j += 2) {
                            const float2 d = fadd2(make_float2(v[j], v[j + 1]), make_float2(nthr, nthr));
                            if (j < 32) {
                                sg0 = __funnelshift_l(__float_as_uint(d.x), sg0, 1);
                                sg0 = __funnelshift_l(__float_as_uint(d.y), sg0, 1);
                            } else {
                                sg1 = __funnelshift_l(__float_as_uint(d.x), sg1, 1);
                                sg1 = __funnelshift_l(__float_as_uint(d.y), sg1, 1);
                            }
                        }
                    }
                    w0 = __brev(~sg0);
                    w1 = __brev(~sg1);
                    if (nvis < 64) {  // invisible keys (causal / ragged tail / row past N_p)
                        w0 &= nvis >= 32 ? 0xffffffffu : ((1u << nvis) - 1u);
                        w1 &= nvis >= 64 ? 0xffffffffu : (nvis <= 32 ? 0u : ((1u << (nvis - 32)) - 1u));
                    }
                } else if constexpr (EPI == EPI_MAX) {
                    if (nvis < 64) {
#pragma unroll
                        for (int j = 0; j < 64; ++j)
                            if (j >= nvis) v[j] = -INFINITY;
                    }
                    float a = -INFINITY, b = -INFINITY, c2 = -INFINITY, d2 = -INFINITY;  // 4 chains
#pragma unroll
                    for (int j = 0; j < 64; j += 8) {
                        a = fmax3(a, v[j], v[j + 1]);
                        b = fmax3(b, v[j + 2], v[j + 3]);
                        c2 = fmax3(c2, v[j + 4], v[j + 5]);
                        d2 = fmax3(d2, v[j + 6], v[j + 7]);
                    }
                    m_run = fmaxf(m_run, fmaxf(fmaxf(a, b), fmaxf(c2, d2)));
                } else if constexpr (EPI == EPI_THRESH) {
                    // keep = s >= thr <=> sign bit of s - thr clear (see EPI_ALG1)
                    const float nthr = -thr_fixed;
                    uint32_t sg0 = 0u, sg1 = 0u;
#pragma unroll
                    for (int j = 0; j < 32; j += 2) {
                        const float2 d0 = fadd2(make_float2(v[j], v[j + 1]), make_float2(nthr, nthr));
                        const float2 d1 = fadd2(make_float2(v[32 + j], v[32 + j + 1]), make_float2(nthr, nthr));
                        sg0 = __funnelshift_l(__float_as_uint(d0.x), sg0, 1);
                        sg0 = __funnelshift_l(__float_as_uint(d0.y), sg0, 1);
                        sg1 = __funnelshift_l(__float_as_uint(d1.x), sg1, 1);
                        sg1 = __funnelshift_l(__float_as_uint(d1.y), sg1, 1);
                    }
                    w0 = __brev(~sg0);
                    w1 = __brev(~sg1);
                    if (nvis < 64) {
                        w0 &= nvis >= 32 ? 0xffffffffu : ((1u << nvis) - 1u);
                        w1 &= nvis >= 64 ? 0xffffffffu : (nvis <= 32 ? 0u : ((1u << (nvis - 32)) - 1u));
                    }
                } else if constexpr (EPI == EPI_TK_MINMAX) {
                    float a = -INFINITY, b2 = -INFINITY, c2 = INFINITY, d2 = INFINITY;
                    if (nvis == 64) {
#pragma unroll
                        for (int j = 0; j < 64; j += 4) {
                            a = fmax3(a, v[j], v[j + 1]);
                            b2 = fmax3(b2, v[j + 2], v[j + 3]);
                            c2 = fminf(fminf(c2, v[j]), v[j + 1]);
                            d2 = fminf(fminf(d2, v[j + 2]), v[j + 3]);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 64; ++j) {
                            if (j < nvis) {
                                a = fmaxf(a, v[j]);
                                c2 = fminf(c2, v[j]);
                            }
                        }
                    }
                    m_run = fmaxf(m_run, fmaxf(a, b2));
                    mn_run = fminf(mn_run, fminf(c2, d2));
                } else if constexpr (EPI == EPI_TK_SHIST) {
                    // bin = round((top - s) * invw): round-to-nearest by the 1.5*2^23 magic add,
                    // the integer read from the mantissa; bins outside [0, 255] are skipped
                    // (level 2 also counts the scores above its range: bin < 0)
                    uint32_t* hcol = hist + r;
#pragma unroll
                    for (int j = 0; j < 64; ++j) {
                        const float t = fmaf(v[j], -tk_b, tk_a) + 12582912.f;
                        const int bi = __float_as_int(t) - 0x4B400000;
                        const uint32_t bin = (uint32_t)bi;
                        if (j < nvis && bin < 256u) atomicAdd(hcol + bin * 128, 1u);
                        if (p.pass == 1) above += (j < nvis && bi < 0) ? 1u : 0u;
                    }
                } else if constexpr (EPI == EPI_TK_CAND) {
                    // above = s > hi, inside = lo <= s <= hi, as sign bits of hi - s and s - lo
                    // (the ALG1 trick; +-inf bounds give +inf differences), then predicated stores
                    uint32_t ab0 = 0u, ab1 = 0u, lo0 = 0u, lo1 = 0u;
#pragma unroll
                    for (int j = 0; j < 32; j += 2) {
                        const float2 ha = fadd2(make_float2(tk_b, tk_b), make_float2(-v[j], -v[j + 1]));
                        const float2 hb = fadd2(make_float2(tk_b, tk_b), make_float2(-v[32 + j], -v[33 + j]));
                        const float2 la = fadd2(make_float2(v[j], v[j + 1]), make_float2(-tk_a, -tk_a));
                        const float2 lb = fadd2(make_float2(v[32 + j], v[33 + j]), make_float2(-tk_a, -tk_a));
                        ab0 = __funnelshift_l(__float_as_uint(ha.x), ab0, 1);
                        ab0 = __funnelshift_l(__float_as_uint(ha.y), ab0, 1);
                        ab1 = __funnelshift_l(__float_as_uint(hb.x), ab1, 1);
                        ab1 = __funnelshift_l(__float_as_uint(hb.y), ab1, 1);
                        lo0 = __funnelshift_l(__float_as_uint(la.x), lo0, 1);
                        lo0 = __funnelshift_l(__float_as_uint(la.y), lo0, 1);
                        lo1 = __funnelshift_l(__float_as_uint(lb.x), lo1, 1);
                        lo1 = __funnelshift_l(__float_as_uint(lb.y), lo1, 1);
                    }
                    const uint32_t vm0 = nvis >= 32 ? 0xffffffffu : ((1u << nvis) - 1u);
                    const uint32_t vm1 = nvis >= 64 ? 0xffffffffu : (nvis <= 32 ? 0u : ((1u << (nvis - 32)) - 1u));
                    ab0 = __brev(ab0) & vm0;
                    ab1 = __brev(ab1) & vm1;
                    const uint32_t in0 = ~(ab0 | __brev(lo0)) & vm0;
                    const uint32_t in1 = ~(ab1 | __brev(lo1)) & vm1;
                    above += __popc(ab0) + __popc(ab1);
                    // extraction: the 64 scores go to a column-major shared stage (conflict-free:
                    // lanes are consecutive rows), then each thread walks its set bits (~4% of
                    // scores) reading the stage with a dynamic index
                    float* stg = reinterpret_cast<float*>(hist) + eset * 64 * 128 + r;
#ifdef VA_TK_CAND_NOSTORE
                    ncand += __popc(in0) + __popc(in1);
                    if (false) {
#else
                    if ((in0 | in1) != 0u) {
#endif
#pragma unroll
                        for (int j = 0; j < 64; ++j) stg[j * 128] = v[j];
                        // candidates go through a 4-entry register buffer and leave as one 16-B
                        // store of scores + one of indices (a quarter of the scattered store
                        // transactions of per-candidate 4-B stores; each lane is its own row)
                        const uint32_t cap = (uint32_t)subcap;
#pragma unroll
                        for (int half = 0; half < 2; ++half) {
                            uint32_t m = half ? in1 : in0;
                            while (m) {
                                const int j = 32 * half + __ffs(m) - 1;
                                m &= m - 1u;
                                if (ncand < cap) {
                                    const float sv = stg[j * 128];
                                    const int32_t si = (int32_t)(kc + j);
                                    cb_v[0] = nb == 0 ? sv : cb_v[0];
                                    cb_v[1] = nb == 1 ? sv : cb_v[1];
                                    cb_v[2] = nb == 2 ? sv : cb_v[2];
                                    cb_v[3] = nb == 3 ? sv : cb_v[3];
                                    cb_i[0] = nb == 0 ? si : cb_i[0];
                                    cb_i[1] = nb == 1 ? si : cb_i[1];
                                    cb_i[2] = nb == 2 ? si : cb_i[2];
                                    cb_i[3] = nb == 3 ? si : cb_i[3];
                                    if (++nb == 4) {
                                        const uint32_t at = ncand - 3u;  // a multiple of 4
                                        if (vec_ok) {
                                            *reinterpret_cast<float4*>(cand_row + at) = make_float4(cb_v[0], cb_v[1], cb_v[2], cb_v[3]);
                                            *reinterpret_cast<int4*>(cidx_row + at) = make_int4(cb_i[0], cb_i[1], cb_i[2], cb_i[3]);
                                        } else {
#pragma unroll
                                            for (int e = 0; e < 4; ++e) {
                                                cand_row[at + e] = cb_v[e];
                                                cidx_row[at + e] = cb_i[e];
                                            }
                                        }
                                        nb = 0;
                                    }
                                }
                                ++ncand;
                            }
                        }
                    }
                    w0 = ab0;  // keys above the window are kept whatever the k-th largest is
                    w1 = ab1;
                } else if constexpr (EPI == EPI_TOPK_HIST) {
                    // branch-free: invisible keys are masked by a predicate, the prefix test of
                    // passes > 0 and the histogram update are predicated shared-memory atomics
                    const int pass = p.pass;
                    const bool all = pass == 0;
                    const uint32_t sh_pre = (uint32_t)(32 - 8 * pass) & 31u, sh_dig = (uint32_t)(24 - 8 * pass);
                    uint32_t* hcol = hist + r;
#pragma unroll
                    for (int j = 0; j < 64; ++j) {
                        const uint32_t u = f32_order_key(v[j]);
                        const bool match = (j < nvis) && (all || (u >> sh_pre) == tk_prefix);
                        if (match) atomicAdd(hcol + ((u >> sh_dig) & 255u) * 128, 1u);
                    }
                } else if constexpr (EPI == EPI_TOPK_EMIT) {
                    // keep = key above the k-th largest's key, or equal to it while ties remain
                    // (lowest index first).  Strictly-greater and equal keys are bit-packed
                    // branch-free; the rare ties are then taken from the lowest set bits.
                    uint32_t e0 = 0u, e1 = 0u;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t ua = f32_order_key(v[j]), ub = f32_order_key(v[32 + j]);
                        w0 |= (ua > tk_prefix ? 1u : 0u) << j;
                        w1 |= (ub > tk_prefix ? 1u : 0u) << j;
                        e0 |= (ua == tk_prefix ? 1u : 0u) << j;
                        e1 |= (ub == tk_prefix ? 1u : 0u) << j;
                    }
                    const uint32_t vm0 = nvis >= 32 ? 0xffffffffu : ((1u << nvis) - 1u);
                    const uint32_t vm1 = nvis >= 64 ? 0xffffffffu : (nvis <= 32 ? 0u : ((1u << (nvis - 32)) - 1u));
                    w0 &= vm0;
                    w1 &= vm1;
                    e0 &= vm0;
                    e1 &= vm1;
                    while ((e0 | e1) != 0u && tk_taken < tk_krem) {
                        if (e0) {
                            const uint32_t lo = e0 & (0u - e0);
                            w0 |= lo;
                            e0 ^= lo;
                        } else {
                            const uint32_t lo = e1 & (0u - e1);
                            w1 |= lo;
                            e1 ^= lo;
                        }
                        ++tk_taken;
                    }
                }
                words[2 * c] = w0;
                words[2 * c + 1] = w1;
            }
            tc_fence_before();
            mbar_arrive(&acc_empty[buf]);

            if constexpr (EPI == EPI_ALG1 || EPI == EPI_THRESH || EPI == EPI_TOPK_EMIT || EPI == EPI_TK_CAND) {
                if (row_ok && epi_warps<EPI>() == 8) {  // CAND, two warp sets: each stores its 64-key chunk's words
                    uint32_t* dst = p.bitmask + grow * p.words_per_row + key0 / 32 + 2 * eset;
                    *reinterpret_cast<uint2*>(dst) = make_uint2(words[2 * eset], words[2 * eset + 1]);
                } else if (row_ok) {
                    uint32_t* dst = p.bitmask + grow * p.words_per_row + key0 / 32;
#pragma unroll
                    for (int w = 0; w < BN / 32; w += 4) {
                        *reinterpret_cast<uint4*>(dst + w) = make_uint4(words[w], words[w + 1], words[w + 2], words[w + 3]);
                        cnt += __popc(words[w]) + __popc(words[w + 1]) + __popc(words[w + 2]) + __popc(words[w + 3]);
                    }
                }
            }
        }

        if constexpr (EPI == EPI_TOPK_HIST || EPI == EPI_TK_SHIST)
            named_bar_sync(1, 32 * epi_warps<EPI>());  // both sets' updates done
        if (row_ok) {
            if constexpr (EPI == EPI_ALG1 || EPI == EPI_THRESH || EPI == EPI_TOPK_EMIT) {
                if (cnt) atomicAdd(&p.counts[grow], cnt);
            } else if constexpr (EPI == EPI_MAX) {
                if (p.split) p.segmax[grow * p.n_seg + seg] = f32_order_key(m_run);
                else if (m_run > -INFINITY) atomicMax(&p.rowmax[grow], f32_order_key(m_run));
            } else if constexpr (EPI == EPI_TK_MINMAX) {
                if (m_run > -INFINITY) {
                    atomicMax(&p.tk_smax[grow], f32_order_key(m_run));
                    atomicMin(&p.tk_smin[grow], f32_order_key(mn_run));
                }
            } else if constexpr (EPI == EPI_TK_CAND) {
                const uint32_t at = min(ncand, (uint32_t)subcap) - nb;  // the buffered tail
#pragma unroll
                for (int e = 0; e < 3; ++e)
                    if ((uint32_t)e < nb) {
                        cand_row[at + e] = cb_v[e];
                        cidx_row[at + e] = cb_i[e];
                    }
                if (above) atomicAdd(&p.tk_cabove[grow], above);
                p.tk_ncand[grow * 2 * p.n_seg + slice] = ncand;
            } else if constexpr (EPI == EPI_TK_SHIST) {
                if (above) atomicAdd(&p.tk_sabove[grow], above);
                uint32_t* gh = p.tk_hist + ((int64_t)p.pass * p.BH * p.Np + grow) * 256;
                if (p.n_seg == 1) {  // the whole sampled row in this unit: plain 16-B stores, half per warp set
                    for (int bin = 128 * eset; bin < 128 * eset + 128; bin += 4)
                        *reinterpret_cast<uint4*>(gh + bin) = make_uint4(hist[bin * 128 + r], hist[(bin + 1) * 128 + r],
                                                                         hist[(bin + 2) * 128 + r], hist[(bin + 3) * 128 + r]);
                } else {
                    for (int bin = 128 * eset; bin < 128 * eset + 128; ++bin) {
                        const uint32_t hc = hist[bin * 128 + r];
                        if (hc) atomicAdd(gh + bin, hc);
                    }
                }
            } else if constexpr (EPI == EPI_TOPK_HIST) {
                // this key segment's counts -> the row's histogram in global memory (the two
                // warp sets flush half of the bins each; most bins are empty)
                uint32_t* gh = p.tk_hist + grow * 256;
                for (int bin = 128 * eset; bin < 128 * eset + 128; ++bin) {
                    const uint32_t hc = hist[bin * 128 + r];
                    if (hc) atomicAdd(gh + bin, hc);
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

// TOPK: one thread per pooled row after each histogram pass (see launch_topk_pick).
__global__ void __launch_bounds__(256) topk_pick_kernel(const __grid_constant__ SelectParams p) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= p.BH * p.Np) return;
    if (p.only_failed && p.tk_fail[row] == 0u) return;
    const int64_t i = row % p.Np;
    const int64_t vis_end = p.causal ? min(p.N, (i + 1) * (int64_t)p.pq) : p.N;
    uint32_t prefix, krem;
    if (p.pass == 0) {  // k_i = min(topk, visible), or round_half_up(keep_frac * visible) in [1, visible]
        int64_t ki;
        if (p.topk > 0) ki = min(p.topk, vis_end);
        else {
            ki = (int64_t)floor((double)p.keep_frac * (double)vis_end + 0.5);
            ki = max((int64_t)1, min(ki, vis_end));
        }
        prefix = 0;
        krem = (uint32_t)ki;
    } else {
        prefix = p.tk_prefix[row];
        krem = p.tk_krem[row];
    }
    // the bin holding the krem-th largest remaining key (scan from the top)
    const uint32_t* h = p.tk_hist + row * 256;
    uint32_t cum = 0;
    int bin = 255;
    for (; bin > 0; --bin) {
        const uint32_t hc = h[bin];
        if (cum + hc >= krem) break;
        cum += hc;
    }
    p.tk_prefix[row] = (prefix << 8) | (uint32_t)bin;
    p.tk_krem[row] = krem - cum;
}

template <int D, int BN, int STAGES, int EPI, int BK = 16>
static cudaError_t launch_sel_t(const SelectParams& p, cudaStream_t st) {
    using C = SelCfg<D, BN, STAGES, EPI>;
    auto kern = select_kernel<D, BN, STAGES, EPI, BK>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    const int64_t units = p.BH * p.n_mt * p.n_seg;
    if (units <= 0) return cudaSuccess;
    kern<<<(unsigned)units, sel_threads<EPI>(), C::kSmem, st>>>(p);
    return cudaGetLastError();
}

template <int D>
static cudaError_t launch_sel_d(const SelectParams& p, int epi, cudaStream_t st) {
    switch (epi) {
        case EPI_ALG1:
            if (p.bk == 8) return launch_sel_t<D, 256, 3, EPI_ALG1, 8>(p, st);
            if (p.bk == 16) return launch_sel_t<D, 256, 3, EPI_ALG1, 16>(p, st);
            if (p.bk == 32) return launch_sel_t<D, 256, 3, EPI_ALG1, 32>(p, st);
            if (p.bk == 64) return launch_sel_t<D, 256, 3, EPI_ALG1, 64>(p, st);
            if (p.bk == 128) return launch_sel_t<D, 256, 3, EPI_ALG1, 128>(p, st);
            if (p.bk == 256) return launch_sel_t<D, 256, 3, EPI_ALG1, 256>(p, st);
            return cudaErrorInvalidValue;
        case EPI_MAX: return launch_sel_t<D, 256, 3, EPI_MAX>(p, st);
        case EPI_THRESH: return launch_sel_t<D, 256, 3, EPI_THRESH>(p, st);
        case EPI_TOPK_HIST: return launch_sel_t<D, 128, 2, EPI_TOPK_HIST>(p, st);
        case EPI_TOPK_EMIT: return launch_sel_t<D, 256, 3, EPI_TOPK_EMIT>(p, st);
        case EPI_SCORES: return launch_sel_t<D, 256, 3, EPI_SCORES>(p, st);
        case EPI_TK_MINMAX: return launch_sel_t<D, 256, 3, EPI_TK_MINMAX>(p, st);
        case EPI_TK_SHIST: return launch_sel_t<D, 128, 2, EPI_TK_SHIST>(p, st);
        case EPI_TK_CAND: return launch_sel_t<D, 128, 2, EPI_TK_CAND>(p, st);
        default: return cudaErrorInvalidValue;
    }
}

int select_bn(int epi) { return (epi == EPI_TOPK_HIST || epi == EPI_TK_SHIST || epi == EPI_TK_CAND) ? 128 : 256; }

cudaError_t launch_select(const SelectParams& p, int epi, int D, cudaStream_t st) {
    if (D == 128) return launch_sel_d<128>(p, epi, st);
    if (D == 64) return launch_sel_d<64>(p, epi, st);
    return cudaErrorInvalidValue;
}

cudaError_t launch_topk_pick(const SelectParams& p, cudaStream_t st) {
    const int64_t R = p.BH * p.Np;
    if (R <= 0) return cudaSuccess;
    topk_pick_kernel<<<(unsigned)((R + 255) / 256), 256, 0, st>>>(p);
    return cudaGetLastError();
}

// ============================================================================ windowed TOPK
// The radix TOPK above needs 4 histogram passes that touch every score (~10 ms each at dit128k).
// Windowed TOPK: estimate the k-th largest score of each row from a 1-in-8 sample of the keys,
// take a window [lo, hi] around it wide enough for the sampling error (c sigma of the binomial
// rank), and make ONE full pass that counts the scores above hi and collects those inside the
// window.  The sample ranks come from two histograms: level 1 (min/max, then 256 bins) on a
// 1-in-64 sub-sample places the value range of level 2 (256 bins + a count of the scores above
// it) on the 1-in-8 sample, wide enough (tk_sigma1 sub-sample sigmas) to hold the window.  The exact k-th largest is then selected
// among the candidates; rows where the window missed it (or overflowed) fall back to the radix
// passes.  The result (tk_prefix = order key of the k-th largest, tk_krem = ties to take) is
// the same state the radix passes produce, so the emit pass and reading R12 are unchanged.

__global__ void tk_sample_k_kernel(const uint4* __restrict__ k, uint4* __restrict__ ks, int64_t BHkv, int64_t N,
                                   int64_t Ns, int64_t D, int stride) {
    const int64_t per_row = D / 8;  // uint4 per row
    const int64_t total = BHkv * Ns * per_row;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = x % per_row, js = (x / per_row) % Ns, bh = x / (per_row * Ns);
        // one key per group of `stride`, at a hashed offset: a fixed offset would sample the same
        // position of every period-`stride` structure of the sequence (video patches are 8 wide)
        const uint32_t hsh = (uint32_t)js * 2654435761u;
        int64_t j = js * stride + (int64_t)((hsh >> 16) % (uint32_t)stride);
        if (j >= N) j = N - 1;
        ks[x] = k[(bh * N + j) * per_row + c];
    }
}

namespace {
VA_DEV int64_t tk_budget(const SelectParams& p, int64_t vis_real) {  // k_i (reading R12)
    int64_t ki;
    if (p.topk > 0) ki = min(p.topk, vis_real);
    else {
        ki = (int64_t)floor((double)p.keep_frac * (double)vis_real + 0.5);
        ki = max((int64_t)1, min(ki, vis_real));
    }
    return ki;
}
}  // namespace

// stage 0: init; 1: level-1 binning over [smin, smax] of the sub-sample; 2 (warp kernel below):
// level-2 range = the level-1 bins holding the sub-sample ranks around the k-th largest;
// 3 (warp kernel): the window [lo, hi] from the level-2 histogram and its above count.
// Bin b of a level covers s with round((top - s) * invw) == b, i.e. s in [top - (b+.5)/invw,
// top - (b-.5)/invw]; boundaries are widened by a relative 2^-16 (the exact counts of the
// candidate pass decide, so a wider window only costs candidates).
__global__ void __launch_bounds__(256) tk_rows_kernel(const __grid_constant__ SelectParams p, int stage) {
    const int64_t R = p.BH * p.Np;
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= R) return;
    if (stage == 0) {
        p.tk_smax[row] = 0u;
        p.tk_smin[row] = 0xFFFFFFFFu;
        p.tk_fail[row] = 0u;
        p.tk_cabove[row] = 0u;
        p.tk_sabove[row] = 0u;
        return;
    }
    // stage 1: level-1 binning over the sub-sample's [min, max]: bin = round((top - s) * invw)
    const float smax = f32_from_order_key(p.tk_smax[row]), smin = f32_from_order_key(p.tk_smin[row]);
    const float w = smax - smin;
    p.tk_top[row] = smax;
    p.tk_invw[row] = w > 0.f ? 255.f / w : 0.f;
}

// Stages 2 and 3 of tk_rows_kernel with one warp per row: the histogram walks become warp
// scans (lane l owns 8 consecutive bins; coalesced reads), same arithmetic and the same window.
// Counts are doubled so that the half pieces of stage 3 stay integers.
struct TkScan {
    int hit_lo, hit_hi;  // first index whose running count reaches T_lo / T_hi in this segment, or -1
    uint32_t total;      // doubled counts of the segment
};
// segment a[s0 .. s0 + n) (n <= 256) with doubled counts, running doubled count cum2 before it
VA_DEV TkScan tk_warp_scan(const uint32_t* a, int s0, int n, uint32_t cum2, double t_lo, double t_hi, int lane) {
    uint32_t vv[8];
    uint32_t own = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int x = 8 * lane + t;
        vv[t] = x < n ? 2u * a[s0 + x] : 0u;
        own += vv[t];
    }
    uint32_t incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    TkScan r;
    r.total = __shfl_sync(0xffffffffu, incl, 31);
    const double base = (double)cum2;
    const uint32_t excl = incl - own;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
        const double T = which ? t_hi : t_lo;
        const unsigned ball = __ballot_sync(0xffffffffu, base + (double)incl >= T);
        int hit = -1;
        if (ball) {
            const int L = __ffs(ball) - 1;
            int loc = 7;
            double c = base + (double)excl;
            for (int t = 0; t < 8; ++t) {
                c += (double)vv[t];
                if (c >= T) {
                    loc = t;
                    break;
                }
            }
            hit = 8 * L + __shfl_sync(0xffffffffu, loc, L);
        }
        if (which) r.hit_hi = hit;
        else r.hit_lo = hit;
    }
    return r;
}

__global__ void __launch_bounds__(256) tk_rows_warp_kernel(const __grid_constant__ SelectParams p, int stage, int stride) {
    const int64_t R = p.BH * p.Np;
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (row >= R) return;
    const int64_t i = row % p.Np;
    const int64_t vis_real = p.causal ? min(p.N_real, (i + 1) * (int64_t)p.pq) : p.N_real;
    const int64_t ns = (vis_real + stride - 1) / stride;  // visible keys of this sample
    const double ki = (double)tk_budget(p, vis_real);
    const double ks = ki * (double)ns / (double)vis_real;  // the k-th largest's rank in the sample
    const double pr = min(1.0, ki / (double)vis_real);
    const double sig = sqrt((double)ns * pr * (1.0 - pr));
    if (stage == 2) {
        // sub-sample ranks [ks - d1, ks + d1], d1 = tk_sigma1 sigma + 8: wide enough that the
        // values at the 1-in-8 sample's window ranks fall inside w.h.p. (both samples' errors)
        const double d1 = (double)p.tk_sigma1 * sig + 8.0;
        const uint32_t* h1 = p.tk_hist + row * 256;
        const float smax = f32_from_order_key(p.tk_smax[row]), smin = f32_from_order_key(p.tk_smin[row]);
        const float top1 = smax, invw1 = (smax - smin) > 0.f ? 255.f / (smax - smin) : 0.f;
        // doubled counts against doubled thresholds (tk_warp_scan's convention)
        const TkScan sc = tk_warp_scan(h1, 0, 256, 0u, 2.0 * (ks - d1), 2.0 * (ks + d1), lane);
        const int ba = sc.hit_lo < 0 ? 255 : sc.hit_lo;
        const int bb = sc.hit_hi < 0 ? 255 : sc.hit_hi;
        if (lane == 0) {
            // level-2 range: level-1 bins ba..bb as 256 sub-bins (sub-bin 0 starts at bin ba's top)
            const float top2 = invw1 > 0.f ? top1 - ((float)ba - 0.5f) / invw1 : top1;
            const float invw2 = invw1 > 0.f ? invw1 * 256.f / (float)(bb - ba + 1) : 0.f;
            p.tk_top[row] = top2;
            p.tk_invw[row] = invw2;
        }
        return;
    }
    // stage 3: walk the 1-in-8 sample from the top: the scores above the level-2 range, then its
    // 256 sub-bins; hi = upper edge of the piece holding rank r_lo, lo = lower edge of the piece
    // holding r_hi (-inf when r_hi lies below the range, +inf when r_lo lies above it)
    const double d = (double)p.tk_sigma * sig + 8.0;
    const double r_lo = ks - d, r_hi = ks + d;
    const uint32_t* h2 = p.tk_hist + (R + row) * 256;
    const float top2 = p.tk_top[row], invw2 = p.tk_invw[row];
    float hi = INFINITY, lo = -INFINITY;
    if (invw2 > 0.f) {
        const uint32_t ab2 = 2u * p.tk_sabove[row];
        const double T_hi = 2.0 * r_lo, T_lo = 2.0 * r_hi;  // doubled counts
        const bool hi_in_above = r_lo < 1.0 || (double)ab2 >= T_hi;
        const bool lo_in_above = (double)ab2 >= T_lo;
        if (lo_in_above) {
            lo = top2 + 0.5f / invw2;  // the whole window lies above the range (hi = +inf)
        } else {
            const TkScan sc = tk_warp_scan(h2, 0, 256, ab2, T_hi, T_lo, lane);
            if (!hi_in_above && sc.hit_lo >= 0) hi = top2 - ((float)sc.hit_lo - 0.5f) / invw2;
            if (sc.hit_hi >= 0) lo = top2 - ((float)sc.hit_hi + 0.5f) / invw2;
        }
    }
    if (lane == 0) {
        const float e = 1.0f / 65536.0f;
        p.tk_hi[row] = hi == INFINITY ? INFINITY : hi + fabsf(hi) * e + 1e-30f;
        p.tk_lo[row] = lo == -INFINITY ? -INFINITY : lo - fabsf(lo) * e - 1e-30f;
    }
}

// One warp per row: exact k'-th largest (k' = k - #above) among the window candidates, then
// the kept candidates' bits: key > theta, and the k_rem lowest-index keys == theta (R12).
// Candidates are in slices (candidate-pass segment x warp set), so ties are ranked by index
// explicitly.
//   fast path: every candidate's order key lies in [klo, khi], where the window is locally
//     ~uniform, so ONE histogram pass with linear bins over that range (the top 8 significant
//     bits of key - klo) leaves ~n/200 candidates in the bin holding the k'-th largest; those
//     are ranked exactly by (key desc, index asc) in shared memory (R12's order).
//   radix path (the bin holds > kTkBinCap candidates, e.g. mass ties): radix select on order
//     keys (8-bit digits, warp-private shared histogram) from the first digit where klo and
//     khi differ.
constexpr int kTkMaxTies = 1024;
constexpr uint32_t kTkBinCap = 512;  // fast path: candidates of the k'-th largest's bin
__device__ __forceinline__ int tk_pick_bin(const uint32_t* h, uint32_t krem, int lane, uint32_t& cum) {
    // from the top: lane l owns bins [255 - 8l - 7, 255 - 8l]; returns the bin where the
    // running count from the top reaches krem, cum = count strictly above it
    uint32_t own = 0;
    for (int t = 0; t < 8; ++t) own += h[255 - 8 * lane - t];
    uint32_t incl = own;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - own;
    const unsigned ball = __ballot_sync(0xffffffffu, incl >= krem);
    const int L = __ffs(ball) - 1;
    cum = __shfl_sync(0xffffffffu, excl, L);
    int bin = 255 - 8 * L;
    for (int t = 0; t < 8; ++t, --bin) {
        const uint32_t hc = h[bin];
        if (cum + hc >= krem) break;
        cum += hc;
    }
    return bin;
}

__global__ void __launch_bounds__(256) tk_exact_kernel(const __grid_constant__ SelectParams p) {
    __shared__ uint32_t hist[8][256];
    __shared__ int32_t tie_idx[8][kTkMaxTies];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * 8 + wid;
    if (row >= p.BH * p.Np) return;
    const int64_t i = row % p.Np;
    const int64_t vis_real = p.causal ? min(p.N_real, (i + 1) * (int64_t)p.pq) : p.N_real;
    const int64_t ki = tk_budget(p, vis_real);
    const int64_t nsl = 2 * p.n_seg;  // slices
    const int64_t subcap = p.cand_cap / nsl;
    int64_t n = 0;
    bool over = false;
    for (int64_t sg = 0; sg < nsl; ++sg) {
        const int64_t c = p.tk_ncand[row * nsl + sg];
        n += c;
        over |= c > subcap;
    }
    const int64_t above = p.tk_cabove[row];
    if (!(above < ki && ki <= above + n && !over)) {
        if (lane == 0) {
            p.tk_fail[row] = 1u;
            atomicAdd(p.tk_nfail, 1);
        }
        return;
    }
    const float* cand = p.tk_cand + row * p.cand_cap;
    const int32_t* cidx = p.tk_cidx + row * p.cand_cap;
    uint32_t krem = (uint32_t)(ki - above);
    uint32_t* h = hist[wid];
    uint32_t* bm = p.bitmask + row * p.words_per_row;
    int32_t* tl = tie_idx[wid];
    const uint32_t klo = f32_order_key(p.tk_lo[row]), khi = f32_order_key(p.tk_hi[row]);

    // ---------------------------------------------------------------- fast path
    const uint32_t W = khi - klo;
    const int shb = max(0, (32 - __clz((int)W)) - 8);  // (key - klo) >> shb < 256
    for (int bin = lane; bin < 256; bin += 32) h[bin] = 0u;
    __syncwarp();
    for (int64_t sg = 0; sg < nsl; ++sg) {
        const int64_t c = p.tk_ncand[row * nsl + sg];
        const float* cs = cand + sg * subcap;
        for (int64_t x = lane; x < c; x += 32) {
            const uint32_t d = min(f32_order_key(cs[x]) - klo, W);
            atomicAdd(&h[d >> shb], 1u);
        }
    }
    __syncwarp();
    uint32_t cum;
    const int bb = tk_pick_bin(h, krem, lane, cum);
    const uint32_t m = h[bb];
    __syncwarp();
    if (m <= kTkBinCap) {
        const uint32_t kb = krem - cum;  // to take from bin bb (1 <= kb <= m)
        uint32_t* tu = reinterpret_cast<uint32_t*>(tl + kTkBinCap);
        uint32_t nm = 0;
        for (int64_t sg = 0; sg < nsl; ++sg) {
            const int64_t c = p.tk_ncand[row * nsl + sg];
            const float* cs = cand + sg * subcap;
            const int32_t* is = cidx + sg * subcap;
            for (int64_t x0 = 0; x0 < c; x0 += 32) {
                const int64_t x = x0 + lane;
                const uint32_t u = x < c ? f32_order_key(cs[x]) : 0u;
                const int bin = x < c ? (int)(min(u - klo, W) >> shb) : -1;
                if (bin > bb) {
                    const int32_t key = is[x];
                    atomicOr(&bm[key >> 5], 1u << (key & 31));
                }
                const bool inb = bin == bb;
                const unsigned tb = __ballot_sync(0xffffffffu, inb);
                if (inb) {
                    const uint32_t slot = nm + __popc(tb & ((1u << lane) - 1u));
                    tl[slot] = is[x];
                    tu[slot] = u;
                }
                nm += __popc(tb);
            }
        }
        __syncwarp();
        // rank in (key desc, index asc); the kb first are kept.  theta = key of rank kb - 1.
        for (uint32_t t = lane; t < nm; t += 32) {
            const uint32_t ut = tu[t];
            const int32_t it = tl[t];
            uint32_t rank = 0;
            for (uint32_t o = 0; o < nm; ++o) {
                const uint32_t uo = tu[o];
                rank += (uo > ut || (uo == ut && tl[o] < it)) ? 1u : 0u;
            }
            if (rank < kb) atomicOr(&bm[it >> 5], 1u << (it & 31));
            if (rank == kb - 1) p.tk_prefix[row] = ut;
        }
        if (lane == 0) {
            p.tk_krem[row] = 0u;  // unused downstream on this path
            p.counts[row] = (unsigned long long)ki;  // top-k keeps exactly k_i keys
        }
        return;
    }

    // ---------------------------------------------------------------- radix path
    // every candidate lies in [lo, hi]: the leading bytes their order keys share with both
    // bounds are known, so the radix starts at the first byte where the bounds differ
    int first = 0;
    while (first < 3 && (klo >> (24 - 8 * first)) == (khi >> (24 - 8 * first))) ++first;
    uint32_t prefix = first > 0 ? (klo >> (32 - 8 * first)) : 0u;
    for (int pass = first; pass < 4; ++pass) {
        for (int bin = lane; bin < 256; bin += 32) h[bin] = 0u;
        __syncwarp();
        const int sh = 24 - 8 * pass;
        for (int64_t sg = 0; sg < nsl; ++sg) {
            const int64_t c = p.tk_ncand[row * nsl + sg];
            const float* cs = cand + sg * subcap;
            for (int64_t x = lane; x < c; x += 32) {
                const uint32_t u = f32_order_key(cs[x]);
                if (pass == 0 || (u >> (sh + 8)) == prefix) atomicAdd(&h[(u >> sh) & 255u], 1u);
            }
        }
        __syncwarp();
        const int bin = tk_pick_bin(h, krem, lane, cum);
        prefix = (prefix << 8) | (uint32_t)bin;
        krem -= cum;
        __syncwarp();
    }
    // kept candidates -> bitmask (the keys above the window were set by the candidate pass);
    // ties (key == theta) are gathered and the krem lowest indices kept
    uint32_t nt = 0;
    for (int64_t sg = 0; sg < nsl; ++sg) {
        const int64_t c = p.tk_ncand[row * nsl + sg];
        const float* cs = cand + sg * subcap;
        const int32_t* is = cidx + sg * subcap;
        for (int64_t x0 = 0; x0 < c; x0 += 32) {
            const int64_t x = x0 + lane;
            const uint32_t u = x < c ? f32_order_key(cs[x]) : 0u;
            const bool gt = x < c && u > prefix, tie = x < c && u == prefix;
            if (gt) {
                const int32_t key = is[x];
                atomicOr(&bm[key >> 5], 1u << (key & 31));
            }
            const unsigned tb = __ballot_sync(0xffffffffu, tie);
            if (tie) {
                const uint32_t slot = nt + __popc(tb & ((1u << lane) - 1u));
                if (slot < kTkMaxTies) tl[slot] = is[x];
            }
            nt += __popc(tb);
        }
    }
    __syncwarp();
    if (nt > kTkMaxTies) {  // too many ties to rank here: radix fallback for this row
        if (lane == 0) {
            p.tk_fail[row] = 1u;
            atomicAdd(p.tk_nfail, 1);
        }
        return;
    }
    if (nt == krem) {
        for (uint32_t t = lane; t < nt; t += 32) atomicOr(&bm[tl[t] >> 5], 1u << (tl[t] & 31));
    } else {
        // rank of each tie by index among the ties (indices are distinct)
        for (uint32_t t = lane; t < nt; t += 32) {
            const int32_t a = tl[t];
            uint32_t rank = 0;
            for (uint32_t o = 0; o < nt; ++o) rank += tl[o] < a ? 1u : 0u;
            if (rank < krem) atomicOr(&bm[a >> 5], 1u << (a & 31));
        }
    }
    if (lane == 0) {
        p.tk_prefix[row] = prefix;
        p.tk_krem[row] = krem;
        p.counts[row] = (unsigned long long)ki;  // top-k keeps exactly k_i keys
    }
}

cudaError_t launch_tk_sample_k(const void* k, void* ks, int64_t BHkv, int64_t N, int64_t Ns, int64_t D, int stride,
                               cudaStream_t st) {
    const int64_t total = BHkv * Ns * (D / 8);
    if (total <= 0) return cudaSuccess;
    const int64_t nb = (total + 255) / 256;
    const int grid = (int)(nb < 148 * 16 ? nb : 148 * 16);
    tk_sample_k_kernel<<<grid, 256, 0, st>>>(static_cast<const uint4*>(k), static_cast<uint4*>(ks), BHkv, N, Ns, D,
                                             stride);
    return cudaGetLastError();
}

cudaError_t launch_tk_rows(const SelectParams& p, int stage, int stride, cudaStream_t st) {
    const int64_t R = p.BH * p.Np;
    if (R <= 0) return cudaSuccess;
    if (stage >= 2)
        tk_rows_warp_kernel<<<(unsigned)((R + 7) / 8), 256, 0, st>>>(p, stage, stride);
    else
        tk_rows_kernel<<<(unsigned)((R + 255) / 256), 256, 0, st>>>(p, stage);
    return cudaGetLastError();
}

cudaError_t launch_tk_exact(const SelectParams& p, cudaStream_t st) {
    const int64_t R = p.BH * p.Np;
    if (R <= 0) return cudaSuccess;
    tk_exact_kernel<<<(unsigned)((R + 7) / 8), 256, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace va
