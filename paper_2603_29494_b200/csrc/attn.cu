// attn.cu — vector-sparse attention (Eq. 5, Alg. 2) and the dense reference
// (Eq. 1), one persistent tcgen05/TMEM kernel template, sm_100a.
//
// PAPER.md Eq. 5: for query block i,
//     O[I_B(i)] = softmax( Q[I_B(i)] K[Idx(i)]^T / sqrt(D) ) V[Idx(i)]
// computed with FlashAttention-style online softmax over chunks of gathered K/V
// rows (Alg. 2; App. D.2).
//
// B200 design:
//  * tcgen05 M=128 is the full-rate tile; the paper's query block is P_q = 64 rows
//    (P:335).  A CTA tile is therefore 128 query rows = 128/P_q
//    adjacent blocks, processed over the sorted UNION of their index lists
//    (worklist kernel below).  Each union entry carries per-block membership bits;
//    keys outside a row's own Idx(i) get score -inf, so every row computes exactly
//    Eq. 5 for its own block.  For P_q = 128 the union is the block's own list.
//  * K/V rows are gathered with TMA tile::gather4 (4 rows x 128 B per
//    instruction) into 128B-swizzled shared memory, 128 keys per chunk, 3-stage ring.
//  * S = Q K^T (M=128, N=128, K=D) -> TMEM (double-buffered); softmax warps
//    (thread = query row = TMEM lane) apply masks, online max with lazy rescale
//    (threshold 2^8), exp2, write P as bf16 back into TMEM over S; then
//    O += P V with A = P from TMEM and B = V (MN-major) from shared memory.
//  * Persistent CTAs with a dynamic atomic tile scheduler; tiles ordered
//    head-major (K/V of one head stay L2-resident), causal tiles longest-first.
// Degenerate rows (no visible selected key; reading R6): O_r = V_r,
// LSE_r = scale*<q_r,k_r>.
#include "common.cuh"
#include "kernels.cuh"

#include <math.h>

namespace va {

namespace {

constexpr int kAttnThreads = 320;   // w0 sched+Q, w1 MMA, w2-5 softmax, w6-9 K/V loaders
constexpr int kLoadWarps = 4;
constexpr int kStages = 3;
constexpr uint32_t kPad = 0x3FFFFFFFu;   // meta key for padding lanes (sorts last)

template <int D>
struct AttnCfg {
    static constexpr int kCB = D / 64;
    static constexpr int kTileBytes = kCB * 128 * 128;  // 128 rows x D bf16
    static constexpr int kOffQ = 0;
    static constexpr int kOffK = kTileBytes;
    static constexpr int kOffV = kOffK + kStages * kTileBytes;
    static constexpr int kOffMeta = kOffV + kStages * kTileBytes;
    static constexpr int kMetaWords = 128 + 8;          // keys[128], maskA[4], maskB[4]
    static constexpr int kOffBar = kOffMeta + kStages * kMetaWords * 4;
    // barriers
    static constexpr int B_QFULL = 0, B_QEMPTY = 1, B_KFULL = 2, B_KEMPTY = B_KFULL + kStages,
                         B_VFULL = B_KEMPTY + kStages, B_VEMPTY = B_VFULL + kStages,
                         B_MFULL = B_VEMPTY + kStages, B_SFULL = B_MFULL + kStages, B_PFULL = B_SFULL + 2,
                         B_ODONE = B_PFULL + 2, B_OEMPTY = B_ODONE + 1, B_IFULL = B_OEMPTY + 1,
                         B_IEMPTY = B_IFULL + 2, kNumBars = B_IEMPTY + 2;
    static constexpr int kOffItem = kOffBar + kNumBars * 8;
    static constexpr int kSmem = kOffItem + 16;
    static constexpr uint32_t kTmemCols = 512;          // S0 [0,128) S1 [128,256) O [256,256+D)
    static constexpr uint32_t kIdescS = make_idesc_bf16(128, 128, 0, 0);
    static constexpr uint32_t kIdescPV = make_idesc_bf16(128, D, 0, 1);
};

struct Item {
    int64_t bh, mt;
    int n_chunks;
    int len;       // gather: union length
    int64_t base;  // gather: worklist base
};

template <bool GATHER>
VA_DEV Item decode_item(const AttnParams& p, int item) {
    Item it;
    it.bh = item / p.n_mt;
    it.mt = p.n_mt - 1 - (item % p.n_mt);  // longest-first within a head (causal)
    if constexpr (GATHER) {
        const int64_t G = 128 / p.pq;
        it.len = p.wl_len[it.bh * p.n_mt + it.mt];
        it.base = p.offsets[it.bh * p.Np + G * it.mt];
        it.n_chunks = (it.len + 127) / 128;
    } else {
        const int64_t kend = p.causal ? min(p.N, (it.mt + 1) * 128) : p.N;
        it.len = (int)kend;
        it.base = 0;
        it.n_chunks = (int)((kend + 127) / 128);
    }
    return it;
}

}  // namespace

template <int D, bool GATHER>
__global__ void __launch_bounds__(kAttnThreads, 1) attn_kernel(const __grid_constant__ AttnParams p) {
    using C = AttnCfg<D>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sQ = smem + C::kOffQ;
    uint8_t* sK = smem + C::kOffK;
    uint8_t* sV = smem + C::kOffV;
    uint32_t* sMeta = reinterpret_cast<uint32_t*>(smem + C::kOffMeta);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    int* item_slot = reinterpret_cast<int*>(smem + C::kOffItem);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffItem + 8);

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();

    if (threadIdx.x == 0) {
        if ((smem_u32(smem) & 1023u) != 0) __trap();
        mbar_init(&bars[C::B_QFULL], 1);
        mbar_init(&bars[C::B_QEMPTY], 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars[C::B_KFULL + s], GATHER ? kLoadWarps : 1);
            mbar_init(&bars[C::B_KEMPTY + s], 1);
            mbar_init(&bars[C::B_VFULL + s], GATHER ? kLoadWarps : 1);
            mbar_init(&bars[C::B_VEMPTY + s], 1);
            mbar_init(&bars[C::B_MFULL + s], kLoadWarps);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars[C::B_SFULL + s], 1);
            mbar_init(&bars[C::B_PFULL + s], 128);
            mbar_init(&bars[C::B_IFULL + s], 1);
            mbar_init(&bars[C::B_IEMPTY + s], 1 + 128 + kLoadWarps);
        }
        mbar_init(&bars[C::B_ODONE], 1);
        mbar_init(&bars[C::B_OEMPTY], 128);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t tmem_O = tmem_base + 256;

    if (warp == 0) {
        // ============================================ scheduler: dynamic items + Q tile loads
        if (lane == 0) {
            tma_prefetch_desc(&p.tm_q);
            tma_prefetch_desc(&p.tm_k);
            tma_prefetch_desc(&p.tm_v);
        }
        int qi = 0;  // Q loads issued
        for (int it = 0;; ++it) {
            const int slot = it & 1;
            int item = 0;
            if (lane == 0) {
                if (it >= 2) mbar_wait(&bars[C::B_IEMPTY + slot], ((it >> 1) - 1) & 1);
                item = atomicAdd(p.work_counter, 1);
                item_slot[slot] = item < p.total_items ? item : -1;
                mbar_arrive(&bars[C::B_IFULL + slot]);
            }
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item >= p.total_items) break;
            const Item I = decode_item<GATHER>(p, item);
            if (I.n_chunks == 0) continue;
            if (lane == 0) {
                if (qi > 0) mbar_wait(&bars[C::B_QEMPTY], (qi - 1) & 1);
                mbar_arrive_expect_tx(&bars[C::B_QFULL], C::kTileBytes);
#pragma unroll
                for (int cb = 0; cb < C::kCB; ++cb)
                    tma_load_3d(sQ + cb * 128 * 128, &p.tm_q, &bars[C::B_QFULL], cb * 64, (int)(I.mt * 128),
                                (int)I.bh);
            }
            ++qi;
        }
    } else if (warp >= 6) {
        // ============================================ K/V loaders (4 warps)
        // GATHER: warp g owns chunk columns [32g, 32g+32): reads its 32 union entries
        // (prefetched one chunk ahead), publishes keys + membership ballots (mask word g)
        // to the meta ring, and issues 8 K + 8 V tile::gather4 per column block.
        // Dense: warp 6 issues the K/V tile loads.
        const int g = (int)warp - 6;
        int64_t c = 0;
        for (int it = 0;; ++it) {
            const int slot = it & 1;
            mbar_wait(&bars[C::B_IFULL + slot], (it >> 1) & 1);
            const int item = item_slot[slot];
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars[C::B_IEMPTY + slot]);
            if (item < 0) break;
            const Item I = decode_item<GATHER>(p, item);
            if (I.n_chunks == 0) continue;
            const int64_t b = I.bh / p.Hq, h = I.bh % p.Hq;
            const int64_t bh_kv = b * p.Hkv + h / (p.Hq / p.Hkv);
            if constexpr (GATHER) {
                const uint32_t* wlp = p.wl + I.base;
                int pos = 32 * g + (int)lane;
                uint32_t e_cur = pos < I.len ? __ldg(wlp + pos) : 0u;
                for (int j = 0; j < I.n_chunks; ++j, ++c) {
                    const int s = (int)(c % kStages);
                    const int round = (int)(c / kStages);
                    const bool ok = pos < I.len;
                    const int pos_n = pos + 128;
                    const uint32_t e_nxt = (j + 1 < I.n_chunks && pos_n < I.len) ? __ldg(wlp + pos_n) : 0u;
                    const uint32_t key = e_cur & 0x3FFFFFFFu;
                    const int row = (int)(bh_kv * p.N + (ok ? key : 0u));
                    const uint32_t wA = __ballot_sync(0xffffffffu, ok && ((e_cur >> 30) & 1u));
                    const uint32_t wB = __ballot_sync(0xffffffffu, ok && ((e_cur >> 31) & 1u));
                    if (lane == 0 && round > 0) {
                        mbar_wait(&bars[C::B_KEMPTY + s], (round - 1) & 1);
                        mbar_wait(&bars[C::B_VEMPTY + s], (round - 1) & 1);
                    }
                    __syncwarp();
                    uint32_t* meta = sMeta + s * C::kMetaWords;
                    meta[32 * g + lane] = ok ? key : kPad;
                    if (lane == 0) {
                        meta[128 + g] = wA;
                        meta[132 + g] = wB;
                    }
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(&bars[C::B_MFULL + s]);
                        mbar_arrive_expect_tx(&bars[C::B_KFULL + s], 32 * D * 2);
                        mbar_arrive_expect_tx(&bars[C::B_VFULL + s], 32 * D * 2);
                    }
                    const int r0 = __shfl_sync(0xffffffffu, row, (4 * lane) & 31);
                    const int r1 = __shfl_sync(0xffffffffu, row, (4 * lane + 1) & 31);
                    const int r2 = __shfl_sync(0xffffffffu, row, (4 * lane + 2) & 31);
                    const int r3 = __shfl_sync(0xffffffffu, row, (4 * lane + 3) & 31);
                    __syncwarp();
                    if (lane < 8) {
                        uint8_t* dK = sK + s * C::kTileBytes + (32 * g + 4 * lane) * 128;
                        uint8_t* dV = sV + s * C::kTileBytes + (32 * g + 4 * lane) * 128;
#pragma unroll
                        for (int cb = 0; cb < C::kCB; ++cb)
                            tma_gather4(dK + cb * 128 * 128, &p.tm_k, &bars[C::B_KFULL + s], cb * 64, r0, r1, r2, r3);
#pragma unroll
                        for (int cb = 0; cb < C::kCB; ++cb)
                            tma_gather4(dV + cb * 128 * 128, &p.tm_v, &bars[C::B_VFULL + s], cb * 64, r0, r1, r2, r3);
                    }
                    e_cur = e_nxt;
                    pos = pos_n;
                }
            } else {
                for (int j = 0; j < I.n_chunks; ++j, ++c) {
                    if (g != 0 || lane != 0) continue;
                    const int s = (int)(c % kStages);
                    const int round = (int)(c / kStages);
                    if (round > 0) {
                        mbar_wait(&bars[C::B_KEMPTY + s], (round - 1) & 1);
                        mbar_wait(&bars[C::B_VEMPTY + s], (round - 1) & 1);
                    }
                    uint8_t* dK = sK + s * C::kTileBytes;
                    uint8_t* dV = sV + s * C::kTileBytes;
                    mbar_arrive_expect_tx(&bars[C::B_KFULL + s], C::kTileBytes);
#pragma unroll
                    for (int cb = 0; cb < C::kCB; ++cb)
                        tma_load_3d(dK + cb * 128 * 128, &p.tm_k, &bars[C::B_KFULL + s], cb * 64, j * 128,
                                    (int)bh_kv);
                    mbar_arrive_expect_tx(&bars[C::B_VFULL + s], C::kTileBytes);
#pragma unroll
                    for (int cb = 0; cb < C::kCB; ++cb)
                        tma_load_3d(dV + cb * 128 * 128, &p.tm_v, &bars[C::B_VFULL + s], cb * 64, j * 128,
                                    (int)bh_kv);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // ==================================================================== MMA issuer
        if (elect_one()) {
            int64_t c = 0;
            int qi = 0, oi = 0;
            auto issue_pv = [&](int64_t cc, bool first) {
                const int s = (int)(cc % kStages);
                if (first) {
                    if (oi > 0) mbar_wait(&bars[C::B_OEMPTY], (oi - 1) & 1);
                    ++oi;
                }
                mbar_wait(&bars[C::B_PFULL + (cc & 1)], (uint32_t)((cc >> 1) & 1));
                mbar_wait(&bars[C::B_VFULL + s], (uint32_t)((cc / kStages) & 1));
                tc_fence_after();
                const uint32_t pt = tmem_base + (uint32_t)((cc & 1) * 128);
                const uint32_t va = smem_u32(sV + s * C::kTileBytes);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t bdesc = make_sdesc(va + kk * 16 * 128, 128 * 128, 1024);
                    mma_bf16_ts(tmem_O, pt + kk * 8, bdesc, C::kIdescPV, (first && kk == 0) ? 0u : 1u);
                }
                mma_commit(&bars[C::B_VEMPTY + s]);
                mma_commit(&bars[C::B_ODONE]);
            };
            for (int it = 0;; ++it) {
                const int slot = it & 1;
                mbar_wait(&bars[C::B_IFULL + slot], (it >> 1) & 1);
                const int item = item_slot[slot];
                mbar_arrive(&bars[C::B_IEMPTY + slot]);
                if (item < 0) break;
                const Item I = decode_item<GATHER>(p, item);
                if (I.n_chunks == 0) continue;
                mbar_wait(&bars[C::B_QFULL], qi & 1);
                ++qi;
                tc_fence_after();
                const uint32_t qa = smem_u32(sQ);
                for (int j = 0; j < I.n_chunks; ++j, ++c) {
                    const int s = (int)(c % kStages);
                    mbar_wait(&bars[C::B_KFULL + s], (uint32_t)((c / kStages) & 1));
                    tc_fence_after();
                    const uint32_t ka = smem_u32(sK + s * C::kTileBytes);
                    const uint32_t st = tmem_base + (uint32_t)((c & 1) * 128);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint64_t adesc = make_sdesc(qa + (kk >> 2) * 128 * 128 + (kk & 3) * 32, 16, 1024);
                        const uint64_t bdesc = make_sdesc(ka + (kk >> 2) * 128 * 128 + (kk & 3) * 32, 16, 1024);
                        mma_bf16_ss(st, adesc, bdesc, C::kIdescS, kk > 0 ? 1u : 0u);
                    }
                    mma_commit(&bars[C::B_KEMPTY + s]);
                    mma_commit(&bars[C::B_SFULL + (c & 1)]);
                    if (j == I.n_chunks - 1) mma_commit(&bars[C::B_QEMPTY]);
                    if (j > 0) issue_pv(c - 1, j == 1);
                }
                issue_pv(c - 1, I.n_chunks == 1);
            }
        }
        __syncwarp();
    } else {
        // ==================================================================== softmax / epilogue
        const uint32_t quad = warp & 3u;
        const int r = (int)(quad * 32 + lane);
        const uint32_t lane_off = (quad * 32u) << 16;
        const int member_bit = (p.pq == 64 && r >= 64) ? 31 : 30;
        const float sl2 = p.scale_log2;
        int64_t c = 0;
        for (int it = 0;; ++it) {
            const int slot = it & 1;
            mbar_wait(&bars[C::B_IFULL + slot], (it >> 1) & 1);
            const int item = item_slot[slot];
            mbar_arrive(&bars[C::B_IEMPTY + slot]);
            if (item < 0) break;
            const Item I = decode_item<GATHER>(p, item);
            const int64_t qrow = I.mt * 128 + r;
            const bool row_ok = qrow < p.N;
            float m_ref = -INFINITY;  // log2-domain reference max (lazy rescaling)
            float l = 0.f;
            for (int j = 0; j < I.n_chunks; ++j, ++c) {
                const int s = (int)(c % kStages);
                // visibility mask of the 128 chunk columns for this row
                uint32_t mw[4];
                if constexpr (GATHER) {
                    mbar_wait(&bars[C::B_MFULL + s], (uint32_t)((c / kStages) & 1));
                    const uint32_t* meta = sMeta + s * C::kMetaWords;
#pragma unroll
                    for (int wd = 0; wd < 4; ++wd) mw[wd] = meta[(member_bit == 30 ? 128 : 132) + wd];
                    if (p.causal) {
                        // keys ascending: visible = prefix with key <= qrow
                        int lo = 0, hi = 128;
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            if ((int64_t)meta[mid] <= qrow) lo = mid + 1;
                            else hi = mid;
                        }
#pragma unroll
                        for (int wd = 0; wd < 4; ++wd) {
                            const int nb = lo - 32 * wd;
                            const uint32_t pm = nb >= 32 ? 0xffffffffu : (nb <= 0 ? 0u : ((1u << nb) - 1u));
                            mw[wd] &= pm;
                        }
                    }
                } else {
                    const int64_t key0 = (int64_t)j * 128;
                    const int64_t vend = p.causal ? min(p.N, qrow + 1) : p.N;
                    const int64_t nv = vend - key0;
#pragma unroll
                    for (int wd = 0; wd < 4; ++wd) {
                        const int64_t nb = nv - 32 * wd;
                        mw[wd] = nb >= 32 ? 0xffffffffu : (nb <= 0 ? 0u : ((1u << nb) - 1u));
                    }
                }
                mbar_wait(&bars[C::B_SFULL + (c & 1)], (uint32_t)((c >> 1) & 1));
                tc_fence_after();
                const uint32_t st = tmem_base + lane_off + (uint32_t)((c & 1) * 128);
                const bool full = (mw[0] & mw[1] & mw[2] & mw[3]) == 0xffffffffu;
                __syncwarp();  // reconverge after the per-row causal search (tcgen05.ld is .sync.aligned)
                // ---- pass 1: masked row max, 64 TMEM columns at a time (low register pressure)
                float mx = -INFINITY;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    uint32_t a[32], b[32];
                    tmem_ld32(st + hf * 64, a);
                    tmem_ld32(st + hf * 64 + 32, b);
                    tmem_ld_wait();
                    if (full) {
#pragma unroll
                        for (int t = 0; t < 32; t += 2) {
                            mx = fmaxf(fmaxf(mx, __uint_as_float(a[t])), __uint_as_float(a[t + 1]));
                            mx = fmaxf(fmaxf(mx, __uint_as_float(b[t])), __uint_as_float(b[t + 1]));
                        }
                    } else {
                        const uint32_t ma = mw[2 * hf], mb = mw[2 * hf + 1];
#pragma unroll
                        for (int t = 0; t < 32; ++t) {
                            const float va_ = (ma & (1u << t)) ? __uint_as_float(a[t]) : -INFINITY;
                            const float vb_ = (mb & (1u << t)) ? __uint_as_float(b[t]) : -INFINITY;
                            mx = fmaxf(fmaxf(mx, va_), vb_);
                        }
                    }
                }
                const float m_new = fmaxf(m_ref, mx * sl2);
                if (j > 0) {  // O must be stable (previous PV done) before a rescale
                    mbar_wait(&bars[C::B_ODONE], (uint32_t)((c - 1) & 1));
                    tc_fence_after();
                }
                // Lazy rescale (only when the max grew by > 2^8): per-row decision, but
                // tcgen05.ld/st are warp-collective (.sync.aligned), so the O update is
                // done by the whole warp whenever any lane needs it (others scale by 1).
                const bool need = m_new > m_ref + 8.0f;
                const float corr = need ? ex2(m_ref - m_new) : 1.0f;
                if (need) {
                    l *= corr;
                    m_ref = m_new;
                }
                if (j > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll
                    for (int g = 0; g < D / 32; ++g) {
                        uint32_t o[32];
                        tmem_ld32(tmem_O + lane_off + g * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int t = 0; t < 32; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * corr);
                        tmem_st32(tmem_O + lane_off + g * 32, o);
                    }
                    tmem_st_wait();
                }
                // ---- pass 2: P = exp2(s*scale*log2e - m), bf16-packed into TMEM over S.
                // Half hf reads S columns [64hf, 64hf+64) and writes P columns [32hf, 32hf+32),
                // which only cover S columns already consumed.
                const float neg_m = (m_ref == -INFINITY) ? 0.f : -m_ref;
                float lsum = 0.f;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    uint32_t a[32], b[32], pk[32];
                    tmem_ld32(st + hf * 64, a);
                    tmem_ld32(st + hf * 64 + 32, b);
                    tmem_ld_wait();
                    const uint32_t ma = full ? 0xffffffffu : mw[2 * hf];
                    const uint32_t mb = full ? 0xffffffffu : mw[2 * hf + 1];
#pragma unroll
                    for (int t = 0; t < 32; t += 2) {
                        float p0 = ex2(fmaf(__uint_as_float(a[t]), sl2, neg_m));
                        float p1 = ex2(fmaf(__uint_as_float(a[t + 1]), sl2, neg_m));
                        float p2 = ex2(fmaf(__uint_as_float(b[t]), sl2, neg_m));
                        float p3 = ex2(fmaf(__uint_as_float(b[t + 1]), sl2, neg_m));
                        p0 = (ma & (1u << t)) ? p0 : 0.f;
                        p1 = (ma & (2u << t)) ? p1 : 0.f;
                        p2 = (mb & (1u << t)) ? p2 : 0.f;
                        p3 = (mb & (2u << t)) ? p3 : 0.f;
                        lsum += (p0 + p1) + (p2 + p3);
                        pk[t >> 1] = pack_bf16x2(p0, p1);
                        pk[16 + (t >> 1)] = pack_bf16x2(p2, p3);
                    }
                    tmem_st32(st + hf * 32, pk);
                }
                l += lsum;
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&bars[C::B_PFULL + (c & 1)]);
            }
            // ---------------------------------------------------------------- epilogue
            if (I.n_chunks > 0) {
                __syncwarp();
                mbar_wait(&bars[C::B_ODONE], (uint32_t)((c - 1) & 1));
                tc_fence_after();
            }
            const float inv = l > 0.f ? 1.f / l : 0.f;
            __nv_bfloat16* orow = p.o + (I.bh * p.N + qrow) * D;
            if (I.n_chunks > 0) {
#pragma unroll
                for (int g = 0; g < D / 32; ++g) {
                    uint32_t ov[32];
                    tmem_ld32(tmem_O + lane_off + g * 32, ov);
                    tmem_ld_wait();
                    if (row_ok && l > 0.f) {
#pragma unroll
                        for (int t = 0; t < 32; t += 8) {
                            uint4 w;
                            w.x = pack_bf16x2(__uint_as_float(ov[t]) * inv, __uint_as_float(ov[t + 1]) * inv);
                            w.y = pack_bf16x2(__uint_as_float(ov[t + 2]) * inv, __uint_as_float(ov[t + 3]) * inv);
                            w.z = pack_bf16x2(__uint_as_float(ov[t + 4]) * inv, __uint_as_float(ov[t + 5]) * inv);
                            w.w = pack_bf16x2(__uint_as_float(ov[t + 6]) * inv, __uint_as_float(ov[t + 7]) * inv);
                            *reinterpret_cast<uint4*>(orow + g * 32 + t) = w;
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(&bars[C::B_OEMPTY]);
            }
            if (row_ok) {
                float lse_v;
                if (l > 0.f) {
                    lse_v = (m_ref + __log2f(l)) * 0.69314718055994531f;
                } else {
                    // degenerate row (reading R6): O_r = V_r, LSE_r = scale*<q_r,k_r>
                    const int64_t b = I.bh / p.Hq, h = I.bh % p.Hq;
                    const int64_t bh_kv = b * p.Hkv + h / (p.Hq / p.Hkv);
                    const __nv_bfloat16* vr = p.v + (bh_kv * p.N + qrow) * D;
                    const __nv_bfloat16* kr = p.k + (bh_kv * p.N + qrow) * D;
                    const __nv_bfloat16* qr = p.q + (I.bh * p.N + qrow) * D;
                    float dot = 0.f;
                    for (int t = 0; t < D; ++t) {
                        orow[t] = vr[t];
                        dot = fmaf(__bfloat162float(qr[t]), __bfloat162float(kr[t]), dot);
                    }
                    lse_v = dot * p.scale;
                }
                if (p.lse) p.lse[I.bh * p.N + qrow] = lse_v;
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

// ------------------------------------------------------------------------ worklist
// One warp per 128-row tile: sorted union of the tile's block index lists with
// membership bits (bit 30 = first block, bit 31 = second block), written at the
// tile's CSR base (|A u B| <= |A| + |B| so it fits in place).
__global__ void __launch_bounds__(256) worklist_kernel(const int64_t* __restrict__ offsets,
                                                       const int32_t* __restrict__ indices,
                                                       uint32_t* __restrict__ wl, int32_t* __restrict__ wl_len,
                                                       int64_t BH, int64_t Np, int64_t n_mt, int32_t pq) {
    const int lane = threadIdx.x & 31;
    const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (tile >= BH * n_mt) return;
    const int64_t bh = tile / n_mt, mt = tile % n_mt;
    const int64_t G = 128 / pq;
    const int64_t ia = mt * G;
    const int64_t ra = bh * Np + ia;
    const int64_t base = offsets[ra];
    const int64_t nA = offsets[ra + 1] - offsets[ra];
    if (G == 1) {
        for (int64_t t = lane; t < nA; t += 32) wl[base + t] = (uint32_t)indices[base + t] | (1u << 30);
        if (lane == 0) wl_len[tile] = (int32_t)nA;
        return;
    }
    const bool hasB = ia + 1 < Np;
    const int64_t offB = hasB ? offsets[ra + 1] : 0;
    const int64_t nB = hasB ? offsets[ra + 2] - offsets[ra + 1] : 0;
    const int32_t* A = indices + base;
    const int32_t* Bl = indices + offB;
    const int INF = 0x7FFFFFFF;
    int64_t pa = 0, pb = 0, out = 0;
    const uint32_t lt = (1u << lane) - 1u;
    while (pa < nA || pb < nB) {
        const int a = (pa + lane < nA) ? A[pa + lane] : INF;
        const int bv = (pb + lane < nB) ? Bl[pb + lane] : INF;
        const int amax = __shfl_sync(0xffffffffu, a, 31);
        const int bmax = __shfl_sync(0xffffffffu, bv, 31);
        const int cut = min(amax, bmax);
        const bool takeA = a != INF && a <= cut;
        const bool takeB = bv != INF && bv <= cut;
        // rank of a in the B window (#b < a), and of b in the A window
        int rA = 0, rB = 0;
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1) {
            const int bq = __shfl_sync(0xffffffffu, bv, rA + st - 1);
            if (bq < a) rA += st;
            const int aq = __shfl_sync(0xffffffffu, a, rB + st - 1);
            if (aq < bv) rB += st;
        }
        {   // final step for rank 31 -> 32
            const int bq = __shfl_sync(0xffffffffu, bv, rA);
            if (rA == 31 && bq < a) rA = 32;
            const int aq = __shfl_sync(0xffffffffu, a, rB);
            if (rB == 31 && aq < bv) rB = 32;
        }
        const int bAt = __shfl_sync(0xffffffffu, bv, rA & 31);
        const int aAt = __shfl_sync(0xffffffffu, a, rB & 31);
        const bool commonA = takeA && rA < 32 && bAt == a;
        const bool commonB = takeB && rB < 32 && aAt == bv;
        const uint32_t cmask = __ballot_sync(0xffffffffu, commonA);
        if (takeA) {
            const int pos = lane + rA - __popc(cmask & lt);
            wl[base + out + pos] = (uint32_t)a | (1u << 30) | (commonA ? (1u << 31) : 0u);
        }
        if (takeB && !commonB) {
            const uint32_t below = rB >= 32 ? 0xffffffffu : ((1u << rB) - 1u);
            const int pos = lane + rB - __popc(cmask & below);
            wl[base + out + pos] = (uint32_t)bv | (1u << 31);
        }
        const int nTA = __popc(__ballot_sync(0xffffffffu, takeA));
        const int nTB = __popc(__ballot_sync(0xffffffffu, takeB));
        out += nTA + nTB - __popc(cmask);
        pa += nTA;
        pb += nTB;
    }
    if (lane == 0) wl_len[tile] = (int32_t)out;
}

cudaError_t launch_worklist(const int64_t* offsets, const int32_t* indices, uint32_t* wl, int32_t* wl_len,
                            int64_t BH, int64_t Np, int64_t n_mt, int32_t pq, cudaStream_t st) {
    const int64_t tiles = BH * n_mt;
    const int64_t blocks = (tiles * 32 + 255) / 256;
    if (blocks <= 0) return cudaSuccess;
    worklist_kernel<<<(unsigned)blocks, 256, 0, st>>>(offsets, indices, wl, wl_len, BH, Np, n_mt, pq);
    return cudaGetLastError();
}

template <int D, bool GATHER>
static cudaError_t launch_attn_t(const AttnParams& p, int grid, cudaStream_t st) {
    using C = AttnCfg<D>;
    auto kern = attn_kernel<D, GATHER>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kAttnThreads, C::kSmem, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_attn(const AttnParams& p, int D, bool gather, int grid, cudaStream_t st) {
    if (D == 128) return gather ? launch_attn_t<128, true>(p, grid, st) : launch_attn_t<128, false>(p, grid, st);
    if (D == 64) return gather ? launch_attn_t<64, true>(p, grid, st) : launch_attn_t<64, false>(p, grid, st);
    return cudaErrorInvalidValue;
}

}  // namespace va
