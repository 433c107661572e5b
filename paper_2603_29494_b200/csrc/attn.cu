// attn.cu — vector-sparse attention (Eq. 5, Alg. 2) and the dense reference
// (Eq. 1): one persistent tcgen05/TMEM kernel template, sm_100a.
//
// PAPER.md Eq. 5: for query block i,
//     O[I_B(i)] = softmax( Q[I_B(i)] K[Idx(i)]^T / sqrt(D) ) V[Idx(i)]
// computed with FlashAttention-style online softmax over chunks of gathered K/V
// rows (Alg. 2; App. D.2).
//
// B200 design (DESIGN.md §6 "attn_kernel"):
//  * Work item = 256 query rows = two M=128 tcgen05 tiles sharing every K/V chunk.
//    The paper's query block is P_q = 64 rows: an item covers
//    256/P_q adjacent blocks.  Its key plan (worklist_kernel / plan_kernel) is the
//    union of their index lists, one membership bit per block (entry = key | bits<<28),
//    in three sorted segments: keys used by both tiles (gathered once, computed by
//    both), by tile 0 only, by tile 1 only.  Softmax is order-invariant, so each row
//    still computes exactly Eq. 5 over its own Idx(i).
//  * Membership masking runs on the tensor core: S = [Q | onehot(block)] [K | bias]^T
//    with one extra K=16 MMA step, bias = 0 (member) or -2^100 (non-member).
//  * 128-key chunks: S_t = Q_t K^T is one M=128 N=128 MMA per K-step (an N=64 MMA with A
//    from shared memory runs at 43% of peak, N=128 at 60%; profiles/ubench_r01.md).
//    TMEM holds O_0, O_1 (128 columns each) and a single S_t buffer per tile (128 columns,
//    P_t written as bf16 over its first 64): per tile the tensor core runs
//    S_t(c) -> [softmax_t] -> PV_t(c) -> S_t(next), and the two tiles ping-pong so each
//    tile's softmax overlaps the other tile's MMAs.  S_t(next) is issued after PV_t(c) (the
//    tensor pipe is in order), so SFULL_t also certifies that O_t is stable for a rescale.
//  * Two ring stages of 128 keys; 4 loader warps, warp (stage s, half h) owns keys
//    [64h, 64h+64) of every chunk on stage s: K_ext rows + K gathers, then the keys for the
//    causal mask + V gathers (TMA tile::gather4, 4 rows x 128 B each); dense mode uses
//    128x64 TMA tiles.
//  * Softmax warpgroup t (thread = query row = TMEM lane): row max over the 128 columns in
//    a first TMEM pass, lazy rescale (threshold 2^8, warp-voted), then exp2 (f32x2 FMA; 1 of
//    4 column groups on the FMA pipe by polynomial) and bf16 P in a second pass.
//  * Persistent CTAs, dynamic atomic scheduler, items head-major (one head's K/V
//    stays L2-resident), causal items longest-first.
// Degenerate rows (no visible selected key; reading R6): O_r = V_r,
// LSE_r = scale*<q_r,k_r>.
#include "common.cuh"
#include "kernels.cuh"
#include "attn_plan.cuh"

#include <math.h>
#include <stdlib.h>

namespace va {

namespace {

// Warpgroups (setmaxnreg works per warpgroup): WG0 = w0 scheduler + Q loads, w1 MMA issuer,
// w2-3 loaders; WG1 = w4-7 softmax tile 0; WG2 = w8-11 softmax tile 1; WG3 = w12-13 loaders
// (w14-15 idle).  The softmax warpgroups raise their register budget to 192 so a thread
// holds its whole 128-column S row; the others drop to 64 (65536 registers in total).
constexpr int kThreads = 512;
constexpr int kLoadWarps = 4;
VA_DEV int loader_index(uint32_t w) { return w == 2 ? 0 : w == 3 ? 1 : w == 12 ? 2 : w == 13 ? 3 : -1; }
VA_DEV void setmaxnreg_inc192() { asm volatile("setmaxnreg.inc.sync.aligned.u32 192;"); }
VA_DEV void setmaxnreg_dec64() { asm volatile("setmaxnreg.dec.sync.aligned.u32 64;"); }
constexpr int kSoftmaxThreads = 256;
constexpr int kChunk = 128;                 // keys per K/V chunk
constexpr uint32_t kKeyMask = 0x0FFFFFFFu;  // entry = key | membership << 28
constexpr uint32_t kPad = 0x0FFFFFFFu;      // meta key for padding lanes (sorts last)
constexpr uint32_t kNegInfBits = 0xff800000u;
// VA_ATTN_ILP (build knob): shorter dependency chains in the softmax (8 max chains, 4 row-sum
// chains).  Sums in a different order: results differ from VA_ATTN_ILP=0 in rounding only.
#ifndef VA_ATTN_ILP
#define VA_ATTN_ILP 1
#endif
#ifndef VA_ATTN_POLY_NUM
#define VA_ATTN_POLY_NUM 1
#endif
#ifndef VA_ATTN_POLY_DEN
#define VA_ATTN_POLY_DEN 4
#endif
#ifndef VA_ATTN_POLY_FAST
#define VA_ATTN_POLY_FAST 0
#endif
// groups g (of 4 columns) with g % kPolyDen < kPolyNum take exp2 on the FMA pipe
constexpr int kPolyNum = VA_ATTN_POLY_NUM, kPolyDen = VA_ATTN_POLY_DEN;

template <int D>
struct AttnCfg {
    static constexpr int kStages = 2;                      // == kLoadWarps / 2 (stage ownership)
    static constexpr int kCB = D / 64;
    static constexpr int kQTileBytes = kCB * 128 * 128;   // 128 rows x D bf16
    static constexpr int kKVBytes = kCB * kChunk * 128;    // 128 keys x D bf16
    static constexpr int kOffQ = 0;                        // two Q tiles
    static constexpr int kOffK = 2 * kQTileBytes;
    static constexpr int kOffV = kOffK + kStages * kKVBytes;
    static constexpr int kOffMeta = kOffV + kStages * kKVBytes;
    static constexpr int kOffQx = (kOffMeta + kStages * kChunk * 4 + 1023) / 1024 * 1024;  // Q_ext [2][128 x 16]
    static constexpr int kOffKx = kOffQx + 2 * 128 * 16 * 2;                               // K_ext [S][128 x 16]
    static constexpr int kOffBar = kOffKx + kStages * kChunk * 16 * 2;
    static constexpr int B_QFULL = 0, B_QEMPTY = 1, B_KFULL = 2, B_KEMPTY = B_KFULL + kStages,
                         B_VFULL = B_KEMPTY + kStages, B_VEMPTY = B_VFULL + kStages,
                         B_MFULL = B_VEMPTY + kStages, B_SFULL = B_MFULL + kStages /* [2 tiles] */,
                         B_PFULL = B_SFULL + 2, B_OEMPTY = B_PFULL + 2, B_OFIN = B_OEMPTY + 2,
                         B_IFULL = B_OFIN + 1, B_IEMPTY = B_IFULL + 2, kNumBars = B_IEMPTY + 2;
    static constexpr int kOffItem = kOffBar + kNumBars * 8;
    static constexpr int kSmem = kOffItem + 16;
    // TMEM: O_t at 128t (D cols); S_t at 256 + 128t (128 cols; P_t over its first 64)
    static constexpr uint32_t kTmemCols = 512;
    static constexpr uint32_t kIdescS = make_idesc_bf16(128, kChunk, 0, 0);
    static constexpr uint32_t kIdescPV = make_idesc_bf16(128, D, 0, 1);
};

VA_DEV uint32_t o_col(int t) { return 128u * t; }
VA_DEV uint32_t s_col(int t) { return 256u + 128u * t; }

using plan::Chunk;
using plan::Item;
using plan::next_chunk;
using plan::trace;
template <bool G>
VA_DEV Item decode_item(const AttnParams& p, int item) { return plan::decode_item<kChunk, G>(p, item); }
template <bool G>
VA_DEV Chunk chunk_info(const Item& I, int j) { return plan::chunk_info<kChunk, G>(I, j); }

}  // namespace

template <int D, bool GATHER>
__global__ void __launch_bounds__(kThreads, 1) attn_kernel(const __grid_constant__ AttnParams p) {
    using C = AttnCfg<D>;
    constexpr int S_ = C::kStages;
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
    if (p.d_nnz != nullptr && *p.d_nnz > p.nnz_cap) return;  // fused path: plan not built (capacity)

    if (threadIdx.x == 0) {
        if ((smem_u32(smem) & 1023u) != 0) __trap();
        mbar_init(&bars[C::B_QFULL], 1);
        mbar_init(&bars[C::B_QEMPTY], 1);
        for (int s = 0; s < S_; ++s) {
            mbar_init(&bars[C::B_KFULL + s], GATHER ? 2 : 1);  // two K half-warps
            mbar_init(&bars[C::B_KEMPTY + s], 1);
            mbar_init(&bars[C::B_VFULL + s], GATHER ? 2 : 1);
            mbar_init(&bars[C::B_VEMPTY + s], 1);
            mbar_init(&bars[C::B_MFULL + s], 2);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&bars[C::B_SFULL + t], 1);
            mbar_init(&bars[C::B_PFULL + t], 128);
            mbar_init(&bars[C::B_OEMPTY + t], 128);
            mbar_init(&bars[C::B_IFULL + t], 1);
            mbar_init(&bars[C::B_IEMPTY + t], 1 + kSoftmaxThreads + kLoadWarps);
        }
        mbar_init(&bars[C::B_OFIN], 1);
        fence_barrier_init();
    }
    if constexpr (GATHER) {
        // Membership masking on the tensor core: S = [Q | E] [K | F]^T with E = one-hot of the
        // row's block (Q_ext, constant per row position) and F[j][b] = 0 if key j is in block
        // b's index set else -2^100 (K_ext, written per chunk by the loaders).  Members get
        // +0 exactly; non-members a score of -2^100 whose exp2 underflows to 0.
        uint16_t* qx = reinterpret_cast<uint16_t*>(smem + C::kOffQx);
        for (int x = threadIdx.x; x < 2 * 128 * 16; x += kThreads) {
            const int t = x / (128 * 16), r = (x / 16) % 128, e = x % 16;
            const int blk = (128 * t + r) / p.pq;
            qx[(t * 128 * 16 * 2 + k16_offset(r, e)) / 2] = (e == blk) ? 0x3F80u : 0u;  // bf16 1.0
        }
        uint32_t* kx = reinterpret_cast<uint32_t*>(smem + C::kOffKx);
        for (int x = threadIdx.x; x < S_ * kChunk * 16 / 2; x += kThreads) kx[x] = 0u;
        fence_proxy_async();
    }
    if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const bool softmax_wg = warp >= 4 && warp < 12;

    if (!softmax_wg) {
    setmaxnreg_dec64();  // whole warpgroups WG0 / WG3 (setmaxnreg is warpgroup-collective)
    if (warp == 0) {
        // ======================================== scheduler: dynamic items + Q tile loads
        if (lane == 0) {
            tma_prefetch_desc(&p.tm_q);
            tma_prefetch_desc(&p.tm_k);
            tma_prefetch_desc(&p.tm_v);
        }
        int qi = 0;
        const uint64_t pol_stream = l2_evict_first_policy();  // Q is read once: do not displace K/V in L2
        for (int it = 0;; ++it) {
            const int slot = it & 1;
            int item = 0;
            if (lane == 0) {
                if (it >= 2) mbar_wait(&bars[C::B_IEMPTY + slot], ((it >> 1) - 1) & 1);
                item = plan::next_item(p);
                item_slot[slot] = item < p.total_items ? item : -1;
                mbar_arrive(&bars[C::B_IFULL + slot]);
            }
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item >= p.total_items) break;
            const Item I = decode_item<GATHER>(p, item);
            if (I.n_chunks == 0) continue;
            if (lane == 0) {
                if (qi > 0) mbar_wait(&bars[C::B_QEMPTY], (qi - 1) & 1);
                mbar_arrive_expect_tx(&bars[C::B_QFULL], 2 * C::kQTileBytes);
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int cb = 0; cb < C::kCB; ++cb)
                        tma_load_3d_hint(sQ + t * C::kQTileBytes + cb * 128 * 128, &p.tm_q, &bars[C::B_QFULL], cb * 64,
                                         (int)(I.it * 256 + t * 128), (int)I.bh, pol_stream);
            }
            ++qi;
        }
    } else if (loader_index(warp) >= 0) {
        // ======================================== K/V loaders (4 warps)
        // Warp (stage s = g >> 1, half h = g & 1) owns keys [64h, 64h+64) of every chunk on
        // stage s: K_ext rows and K gathers after KEMPTY, then the keys for the causal mask and
        // the V gathers after VEMPTY.  Whole half-chunks per warp keep the per-warp TMA issue
        // (a fixed per-iteration cost plus ~70 clk per gather4) off the critical path
        // (scripts/ubench_gather.cu); each warp waits only on its own stage's EMPTY phases.
        const int g = loader_index(warp);
        const int so = g >> 1, hh = g & 1;
        const int kb = 64 * hh;  // first key of this warp's half
        int64_t c = 0;           // chunks of all previous items
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
            int j = (int)(((int64_t)so - c % S_ + S_) % S_);  // first chunk on stage `so`
            if constexpr (GATHER) {
                const uint32_t* wlp = p.wl + I.base;
                Chunk ch;
                ch.len = 0;
                ch.start = 0;
                if (j < I.n_chunks) ch = chunk_info<true>(I, j);
                uint32_t e0 = kb + (int)lane < ch.len ? __ldcs(wlp + ch.start + kb + lane) : 0u;
                uint32_t e1 = kb + 32 + (int)lane < ch.len ? __ldcs(wlp + ch.start + kb + 32 + lane) : 0u;
                for (; j < I.n_chunks; j += S_) {
                    const int64_t cc = c + j;
                    const int s = (int)(cc % S_);
                    const int round = (int)(cc / S_);
                    Chunk chn;
                    chn.len = 0;
                    chn.start = 0;
                    if (j + S_ < I.n_chunks) chn = chunk_info<true>(I, j + S_);
                    const uint32_t en0 = kb + (int)lane < chn.len ? __ldcs(wlp + chn.start + kb + lane) : 0u;
                    const uint32_t en1 = kb + 32 + (int)lane < chn.len ? __ldcs(wlp + chn.start + kb + 32 + lane) : 0u;
                    const bool ok0 = kb + (int)lane < ch.len, ok1 = kb + 32 + (int)lane < ch.len;
                    const uint32_t key0 = e0 & kKeyMask, key1 = e1 & kKeyMask;
                    const int r0 = (int)(bh_kv * p.N + (ok0 ? key0 : 0u));
                    const int r1 = (int)(bh_kv * p.N + (ok1 ? key1 : 0u));
                    const int q0 = (4 * (int)lane) & 31;
                    const int a0 = __shfl_sync(0xffffffffu, r0, q0), a1 = __shfl_sync(0xffffffffu, r0, q0 + 1);
                    const int a2 = __shfl_sync(0xffffffffu, r0, q0 + 2), a3 = __shfl_sync(0xffffffffu, r0, q0 + 3);
                    const int b0_ = __shfl_sync(0xffffffffu, r1, q0), b1_ = __shfl_sync(0xffffffffu, r1, q0 + 1);
                    const int b2_ = __shfl_sync(0xffffffffu, r1, q0 + 2), b3_ = __shfl_sync(0xffffffffu, r1, q0 + 3);
                    const bool lo = lane < 8;
                    const int ra = lo ? a0 : b0_, rb = lo ? a1 : b1_, rc = lo ? a2 : b2_, rd = lo ? a3 : b3_;
                    // ---- K: bias rows, then the gathers
                    if (round > 0) mbar_wait(&bars[C::B_KEMPTY + s], (round - 1) & 1);  // all lanes: no divergence
                    if (lane == 0 && hh == 0) trace(p, 0, cc);
                    __syncwarp();
                    {
                        // K_ext row: bias 0 for member blocks, -2^100 (bf16 0xF180) otherwise
                        uint8_t* kx = smem + C::kOffKx + s * kChunk * 16 * 2;
                        const uint32_t m0 = ok0 ? (e0 >> 28) : 0u, m1 = ok1 ? (e1 >> 28) : 0u;
                        auto bias = [](uint32_t mem) {
                            const uint32_t x0 = (mem & 1u) ? 0u : 0xF180u, x1 = (mem & 2u) ? 0u : 0xF180u;
                            const uint32_t x2 = (mem & 4u) ? 0u : 0xF180u, x3 = (mem & 8u) ? 0u : 0xF180u;
                            return make_uint4(x0 | (x1 << 16), x2 | (x3 << 16), 0u, 0u);
                        };
                        *reinterpret_cast<uint4*>(kx + k16_offset(kb + (int)lane, 0)) = bias(m0);
                        *reinterpret_cast<uint4*>(kx + k16_offset(kb + 32 + (int)lane, 0)) = bias(m1);
                        fence_proxy_async();  // generic-proxy smem write -> tcgen05.mma (async proxy)
                    }
                    __syncwarp();
                    mbar_arrive_expect_tx_if(&bars[C::B_KFULL + s], 64 * D * 2, lane == 0);
                    if (lane < 16) {
                        uint8_t* dst = sK + s * C::kKVBytes + (kb + 4 * (int)lane) * 128;
#pragma unroll
                        for (int cb = 0; cb < C::kCB; ++cb)
                            tma_gather4(dst + cb * kChunk * 128, &p.tm_k, &bars[C::B_KFULL + s], cb * 64, ra, rb, rc,
                                        rd);
                    }
                    // ---- V: keys for the causal mask, then the gathers
                    if (round > 0) mbar_wait(&bars[C::B_VEMPTY + s], (round - 1) & 1);
                    if (lane == 0 && hh == 0) trace(p, 1, cc);
                    __syncwarp();
                    sMeta[s * kChunk + kb + lane] = ok0 ? key0 : kPad;
                    sMeta[s * kChunk + kb + 32 + lane] = ok1 ? key1 : kPad;
                    __syncwarp();
                    mbar_arrive_if(&bars[C::B_MFULL + s], lane == 0 && p.causal);  // waited by the causal softmax only
                    mbar_arrive_expect_tx_if(&bars[C::B_VFULL + s], 64 * D * 2, lane == 0);
                    if (lane < 16) {
                        uint8_t* dst = sV + s * C::kKVBytes + (kb + 4 * (int)lane) * 128;
#pragma unroll
                        for (int cb = 0; cb < C::kCB; ++cb)
                            tma_gather4(dst + cb * kChunk * 128, &p.tm_v, &bars[C::B_VFULL + s], cb * 64, ra, rb, rc,
                                        rd);
                    }
                    e0 = en0;
                    e1 = en1;
                    ch = chn;
                }
            } else {
                if (lane == 0 && hh == 0) {
                    for (; j < I.n_chunks; j += S_) {
                        const int64_t cc = c + j;
                        const int s = (int)(cc % S_);
                        const int round = (int)(cc / S_);
                        if (round > 0) mbar_wait(&bars[C::B_KEMPTY + s], (round - 1) & 1);
                        mbar_arrive_expect_tx(&bars[C::B_KFULL + s], C::kKVBytes);
#pragma unroll
                        for (int cb = 0; cb < C::kCB; ++cb)
                            tma_load_3d(sK + s * C::kKVBytes + cb * kChunk * 128, &p.tm_k, &bars[C::B_KFULL + s],
                                        cb * 64, j * kChunk, (int)bh_kv);
                        if (round > 0) mbar_wait(&bars[C::B_VEMPTY + s], (round - 1) & 1);
                        mbar_arrive_expect_tx(&bars[C::B_VFULL + s], C::kKVBytes);
#pragma unroll
                        for (int cb = 0; cb < C::kCB; ++cb)
                            tma_load_3d(sV + s * C::kKVBytes + cb * kChunk * 128, &p.tm_v, &bars[C::B_VFULL + s],
                                        cb * 64, j * kChunk, (int)bh_kv);
                    }
                }
                __syncwarp();
            }
            c += I.n_chunks;
        }
    } else if (warp == 1) {
        // ======================================== MMA issuer (single thread)
        // Per item: S_t(first chunk of t) for both tiles; then for every chunk j in order and
        // each tile t of j: PV_t(j) (after softmax_t(j)), then S_t(next chunk of t) -- issued
        // after PV_t(j) because S_t overwrites P_t (in-order tensor pipe) and committed to
        // SFULL_t, which therefore also certifies PV_t(j) complete.
        if (elect_one()) {
            int64_t c = 0;              // chunks of previous items (stage rings)
            uint32_t np_[2] = {0, 0};   // PFULL_t phases consumed
            int qi = 0, oi = 0;
            const uint32_t qa = smem_u32(sQ);
            auto wait_k = [&](int64_t cc) {
                mbar_wait(&bars[C::B_KFULL + (int)(cc % S_)], (uint32_t)((cc / S_) & 1));
                tc_fence_after();
                trace(p, 2, cc);
            };
            auto issue_s = [&](int t, int64_t cc, int kmask) {
                const int s = (int)(cc % S_);
                const uint32_t ka = smem_u32(sK + s * C::kKVBytes);
                const uint32_t q_t = qa + t * C::kQTileBytes;
                const uint32_t st = tmem_base + s_col(t);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint64_t adesc = make_sdesc(q_t + (kk >> 2) * 128 * 128 + (kk & 3) * 32, 16, 1024);
                    const uint64_t bdesc = make_sdesc(ka + (kk >> 2) * kChunk * 128 + (kk & 3) * 32, 16, 1024);
                    mma_bf16_ss(st, adesc, bdesc, C::kIdescS, kk > 0 ? 1u : 0u);
                }
                if constexpr (GATHER) {  // + onehot(block) . bias(key, block)^T (membership mask)
                    const uint64_t adesc = make_sdesc(smem_u32(smem + C::kOffQx + t * 128 * 16 * 2), 128, 256, 0);
                    const uint64_t bdesc = make_sdesc(smem_u32(smem + C::kOffKx + s * kChunk * 16 * 2), 128, 256, 0);
                    mma_bf16_ss(st, adesc, bdesc, C::kIdescS, 1u);
                }
                mma_commit(&bars[C::B_SFULL + t]);
                // K stage free once the last tile reading it has issued its S (tile 1 after tile 0)
                if (t == (kmask == 1 ? 0 : 1)) mma_commit(&bars[C::B_KEMPTY + s]);
            };
            for (int it = 0;; ++it) {
                const int slot = it & 1;
                mbar_wait(&bars[C::B_IFULL + slot], (it >> 1) & 1);
                const int item = item_slot[slot];
                mbar_arrive(&bars[C::B_IEMPTY + slot]);
                if (item < 0) break;
                const Item I = decode_item<GATHER>(p, item);
                const int n = I.n_chunks;
                if (n == 0) continue;
                mbar_wait(&bars[C::B_QFULL], qi & 1);
                ++qi;
                if (oi > 0) {  // O_0 / O_1 of the previous item drained by the epilogues
                    mbar_wait(&bars[C::B_OEMPTY + 0], (oi - 1) & 1);
                    mbar_wait(&bars[C::B_OEMPTY + 1], (oi - 1) & 1);
                }
                ++oi;
                tc_fence_after();
                int nx[2];
                nx[0] = (chunk_info<GATHER>(I, 0).mask & 1) ? 0 : next_chunk<GATHER>(I, 0, 0);
                nx[1] = (chunk_info<GATHER>(I, 0).mask & 2) ? 0 : next_chunk<GATHER>(I, 1, 0);
                bool started[2] = {false, false};
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    if (nx[t] < n) {
                        wait_k(c + nx[t]);
                        issue_s(t, c + nx[t], chunk_info<GATHER>(I, nx[t]).mask);
                    }
                }
                for (int j = 0; j < n; ++j) {
                    const int64_t cc = c + j;
                    const int s = (int)(cc % S_);
                    const int m = chunk_info<GATHER>(I, j).mask;
                    mbar_wait(&bars[C::B_VFULL + s], (uint32_t)((cc / S_) & 1));
                    trace(p, 3, cc);
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        if (!(m & (1 << t))) continue;
                        mbar_wait(&bars[C::B_PFULL + t], np_[t] & 1u);
                        ++np_[t];
                        tc_fence_after();
                        const uint32_t pt = tmem_base + s_col(t);
                        const uint32_t ot = tmem_base + o_col(t);
                        const uint32_t va = smem_u32(sV + s * C::kKVBytes);
#pragma unroll
                        for (int kk = 0; kk < kChunk / 16; ++kk) {
                            const uint64_t bdesc = make_sdesc(va + kk * 16 * 128, kChunk * 128, 1024);
                            mma_bf16_ts(ot, pt + kk * 8, bdesc, C::kIdescPV, (!started[t] && kk == 0) ? 0u : 1u);
                        }
                        started[t] = true;
                        trace(p, 4 + t, cc);
                        const int x = next_chunk<GATHER>(I, t, j);
                        if (x < n) {
                            wait_k(c + x);
                            issue_s(t, c + x, chunk_info<GATHER>(I, x).mask);
                        }
                    }
                    mma_commit(&bars[C::B_VEMPTY + s]);
                }
                mma_commit(&bars[C::B_QEMPTY]);  // Q tiles free (every S of the item issued)
                mma_commit(&bars[C::B_OFIN]);    // every MMA of the item complete
                c += n;
            }
        }
        __syncwarp();
    }
    } else {
        setmaxnreg_inc192();
        // ======================================== softmax / epilogue (two warpgroups)
        const int tile = ((int)warp - 4) >> 2;
        const uint32_t quad = warp & 3u;
        const int r = (int)(quad * 32 + lane);
        const uint32_t lane_off = (quad * 32u) << 16;
        const uint32_t tO = tmem_base + lane_off + o_col(tile);
        const uint32_t tS = tmem_base + lane_off + s_col(tile);
        const int row_in_item = 128 * tile + r;
        const float sl2 = p.scale_log2;
        int64_t c = 0;
        uint32_t ns = 0;  // SFULL_t phases consumed
        uint32_t fi = 0;  // OFIN phases consumed (items with chunks)
        for (int it = 0;; ++it) {
            const int slot = it & 1;
            mbar_wait(&bars[C::B_IFULL + slot], (it >> 1) & 1);
            const int item = item_slot[slot];
            mbar_arrive(&bars[C::B_IEMPTY + slot]);
            if (item < 0) break;
            const Item I = decode_item<GATHER>(p, item);
            const int64_t qrow = I.it * 256 + row_in_item;
            const bool row_ok = qrow < p.N;
            const int64_t qrow_w0 = I.it * 256 + 128 * tile + 32 * quad;  // warp's first row
            float m_ref = -INFINITY;  // log2-domain reference max (lazy rescaling)
            float2 lsum2 = make_float2(0.f, 0.f);
            int jt = 0;  // chunks of this item processed by this tile
            for (int j = 0; j < I.n_chunks; ++j, ++c) {
                const int s = (int)(c % S_);
                const Chunk chk = chunk_info<GATHER>(I, j);
                if (!(chk.mask & (1 << tile))) continue;
                // ---- causal / ragged prefix (per row): visible columns [0, lo)
                bool need_prefix = false;
                int lo = kChunk;
                if constexpr (GATHER) {
                    if (p.causal) {
                        mbar_wait(&bars[C::B_MFULL + s], (uint32_t)((c / S_) & 1));
                        const uint32_t* meta = sMeta + s * kChunk;
                        if ((int64_t)meta[kChunk - 1] > qrow_w0) {  // (padding sorts last)
                            need_prefix = true;
                            int a_ = 0, b_ = kChunk;  // keys ascending: visible = prefix with key <= qrow
                            while (a_ < b_) {
                                const int mid = (a_ + b_) >> 1;
                                if ((int64_t)meta[mid] <= qrow) a_ = mid + 1;
                                else b_ = mid;
                            }
                            lo = a_;
                        }
                    }
                } else {
                    const int64_t k0 = (int64_t)j * kChunk;
                    if (chk.len < kChunk || (p.causal && k0 + kChunk - 1 > qrow_w0)) {
                        need_prefix = true;
                        const int64_t vend = p.causal ? min((int64_t)chk.len, qrow - k0 + 1) : (int64_t)chk.len;
                        lo = (int)max((int64_t)0, min((int64_t)kChunk, vend));
                    }
                }
                need_prefix = __any_sync(0xffffffffu, need_prefix);  // warp-uniform branch below
                mbar_wait(&bars[C::B_SFULL + tile], ns & 1u);
                ++ns;
                tc_fence_after();
                if (lane == 0 && (warp == 4 || warp == 8)) trace(p, 6 + 2 * tile, c);
                __syncwarp();
                // ---- one TMEM pass: the row's 128 S columns -> registers (192-register budget),
                // masked row max, lazy O rescale, P = exp2(s*scale*log2e - m) bf16-packed over
                // S_t's first 64 columns (every S column is already in registers)
                uint32_t a[128];
#pragma unroll
                for (int qd = 0; qd < 4; ++qd) {
                    uint32_t (&aq)[32] = *reinterpret_cast<uint32_t(*)[32]>(a + 32 * qd);
                    tmem_ld32(tS + 32 * qd, aq);
                }
                tmem_ld_wait();
                if (need_prefix) {
#pragma unroll
                    for (int t = 0; t < 128; ++t) a[t] = (t < lo) ? a[t] : kNegInfBits;
                }
                float mx;
                {
#if VA_ATTN_ILP
                    // 8 independent FMNMX3 chains (8 deep) instead of 4 (16 deep): the row max is
                    // on the softmax's critical path
                    float m8[8];
#pragma unroll
                    for (int x = 0; x < 8; ++x) m8[x] = -INFINITY;
#pragma unroll
                    for (int t = 0; t < 128; t += 16) {
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            m8[x] = fmaxf(fmaxf(m8[x], __uint_as_float(a[t + 2 * x])), __uint_as_float(a[t + 2 * x + 1]));
                    }
                    mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
#else
                    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                    for (int t = 0; t < 128; t += 8) {
                        m4[0] = fmaxf(fmaxf(m4[0], __uint_as_float(a[t])), __uint_as_float(a[t + 1]));
                        m4[1] = fmaxf(fmaxf(m4[1], __uint_as_float(a[t + 2])), __uint_as_float(a[t + 3]));
                        m4[2] = fmaxf(fmaxf(m4[2], __uint_as_float(a[t + 4])), __uint_as_float(a[t + 5]));
                        m4[3] = fmaxf(fmaxf(m4[3], __uint_as_float(a[t + 6])), __uint_as_float(a[t + 7]));
                    }
                    mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
#endif
                }
                const float m_new = fmaxf(m_ref, mx * sl2);
                const bool need = m_new > m_ref + 8.0f;
                const float corr = need ? ex2(m_ref - m_new) : 1.0f;
                if (need) {
                    lsum2.x *= corr;
                    lsum2.y *= corr;
                    m_ref = m_new;
                }
                // SFULL_t(c) certifies PV_t of this tile's previous chunk complete: O_t is stable.
                if (jt > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll
                    for (int gq = 0; gq < D / 8; ++gq) {
                        uint32_t o[8];
                        tmem_ld8(tO + gq * 8, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int t = 0; t < 8; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * corr);
                        tmem_st8(tO + gq * 8, o);
                    }
                    tmem_st_wait();
                }
                {
                    const float neg_m = (m_ref == -INFINITY) ? 0.f : -m_ref;
                    const uint64_t sl2x2 = pack_f32x2(sl2, sl2);
                    const uint64_t nmx2 = pack_f32x2(neg_m, neg_m);
#if VA_ATTN_ILP
                    float2 ls[4] = {lsum2, make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#endif
#pragma unroll
                    for (int qd = 0; qd < 4; ++qd) {
                        uint32_t pk[16];
#pragma unroll
                        for (int t0 = 0; t0 < 32; t0 += 4) {
                            const int t = 32 * qd + t0;
                            const float2 xa = unpack_f32x2(
                                ffma2(pack_f32x2(__uint_as_float(a[t]), __uint_as_float(a[t + 1])), sl2x2, nmx2));
                            const float2 xb = unpack_f32x2(
                                ffma2(pack_f32x2(__uint_as_float(a[t + 2]), __uint_as_float(a[t + 3])), sl2x2, nmx2));
                            float p0, p1, p2, p3;
                            if ((t >> 2) % kPolyDen >= kPolyDen - kPolyNum) {  // FMA-pipe exp2 (MUFU offload)
                                const float2 pa = VA_ATTN_POLY_FAST ? ex2_poly2_fast(xa.x, xa.y) : ex2_poly2(xa.x, xa.y);
                                const float2 pb = VA_ATTN_POLY_FAST ? ex2_poly2_fast(xb.x, xb.y) : ex2_poly2(xb.x, xb.y);
                                p0 = pa.x, p1 = pa.y, p2 = pb.x, p3 = pb.y;
                            } else {
                                p0 = ex2(xa.x), p1 = ex2(xa.y), p2 = ex2(xb.x), p3 = ex2(xb.y);
                            }
#if VA_ATTN_ILP
                            ls[qd] = fadd2(ls[qd], fadd2(make_float2(p0, p1), make_float2(p2, p3)));  // 4 chains
#else
                            lsum2 = fadd2(lsum2, fadd2(make_float2(p0, p1), make_float2(p2, p3)));
#endif
                            pk[t0 >> 1] = pack_bf16x2(p0, p1);
                            pk[(t0 >> 1) + 1] = pack_bf16x2(p2, p3);
                        }
                        tmem_st16(tS + 16 * qd, pk);
                    }
#if VA_ATTN_ILP
                    lsum2 = fadd2(fadd2(ls[0], ls[1]), fadd2(ls[2], ls[3]));
#endif
                    tmem_st_wait();
                }
                tc_fence_before();
                mbar_arrive(&bars[C::B_PFULL + tile]);
                if (lane == 0 && (warp == 4 || warp == 8)) trace(p, 7 + 2 * tile, c);
                ++jt;
            }
            // ---------------------------------------------------------------- epilogue
            // rows that only ever saw masked keys: l = 0 (non-members -> -2^100 -> 0), degenerate
            const float l = (m_ref < -0x1p99f * sl2) ? 0.f : lsum2.x + lsum2.y;  // scale-aware: masked = -2^100*sl2
            const float inv = l > 0.f ? 1.f / l : 0.f;
            const plan::ORow orow = plan::o_row<D>(p, I.bh, qrow);
            if (I.n_chunks > 0) {  // every MMA of the item complete (one OFIN phase per item with chunks)
                mbar_wait(&bars[C::B_OFIN], fi & 1u);
                ++fi;
                tc_fence_after();
            }
            if (jt > 0) {
                __syncwarp();
#pragma unroll
                for (int gq = 0; gq < D / 32; ++gq) {
                    uint32_t ov[32];
                    tmem_ld32(tO + gq * 32, ov);
                    tmem_ld_wait();
                    if (row_ok && l > 0.f) {
#pragma unroll
                        for (int t = 0; t < 32; t += 8) {
                            uint4 w4;
                            w4.x = pack_bf16x2(__uint_as_float(ov[t]) * inv, __uint_as_float(ov[t + 1]) * inv);
                            w4.y = pack_bf16x2(__uint_as_float(ov[t + 2]) * inv, __uint_as_float(ov[t + 3]) * inv);
                            w4.z = pack_bf16x2(__uint_as_float(ov[t + 4]) * inv, __uint_as_float(ov[t + 5]) * inv);
                            w4.w = pack_bf16x2(__uint_as_float(ov[t + 6]) * inv, __uint_as_float(ov[t + 7]) * inv);
                            plan::o_store16<D>(p, orow, gq * 32 + t, w4);  // streamed: evict first
                        }
                    }
                }
            }
            if (I.n_chunks > 0) {  // one OEMPTY arrival per item with chunks (even if this tile had none)
                tc_fence_before();
                mbar_arrive(&bars[C::B_OEMPTY + tile]);
            }
            if (row_ok) {
                if (l > 0.f) {
                    if (p.lse) p.lse[I.bh * p.N + qrow] = (m_ref + __log2f(l)) * 0.69314718055994531f;
                } else {
                    // degenerate row (reading R6): O_r = V_r, LSE_r = scale*<q_r,k_r>
                    const int64_t b = I.bh / p.Hq, h = I.bh % p.Hq;
                    const int64_t bh_kv = b * p.Hkv + h / (p.Hq / p.Hkv);
                    const __nv_bfloat16* vr = p.v + (bh_kv * p.N + qrow) * D;
                    const __nv_bfloat16* kr = p.k + (bh_kv * p.N + qrow) * D;
                    const __nv_bfloat16* qr = p.q + (I.bh * p.N + qrow) * D;
                    float dot = 0.f;
                    for (int t = 0; t < D; t += 8) plan::o_store16<D>(p, orow, t, *reinterpret_cast<const uint4*>(vr + t));
                    for (int t = 0; t < D; ++t) dot = fmaf(__bfloat162float(qr[t]), __bfloat162float(kr[t]), dot);
                    if (p.lse) p.lse[I.bh * p.N + qrow] = dot * p.scale;
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

// ------------------------------------------------------------------------ worklist
// One CTA per 256-row item (G = 256/P_q blocks; tile 0 = blocks [0, G/2), tile 1 = the
// rest).  Builds the sorted union of the item's block index lists with one membership
// bit per block (entry = key | bits << 28), split into three segments -- keys used by
// both tiles, by tile 0 only, by tile 1 only -- written back to back at the item's CSR
// base (|union| <= sum of list lengths, so it fits in place); wl_len[3*item + {0,1,2}]
// receives the segment lengths.  Per-block bitmaps in shared memory (atomicOr), then a
// block-wide scan of per-word popcounts; key stripes of kStripe keys, with a counting
// pre-pass when N > kStripe.
constexpr int kWlThreads = 512;
constexpr int kStripe = 262144;
constexpr int kStripeWords = kStripe / 32;

struct Seg3 {
    int b, o0, o1;
};

__device__ __forceinline__ Seg3 block_scan3(Seg3 v, Seg3* tot_out, int* sh /* [3][16] */) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    Seg3 inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int nb = __shfl_up_sync(0xffffffffu, inc.b, o);
        const int n0 = __shfl_up_sync(0xffffffffu, inc.o0, o);
        const int n1 = __shfl_up_sync(0xffffffffu, inc.o1, o);
        if (lane >= o) {
            inc.b += nb;
            inc.o0 += n0;
            inc.o1 += n1;
        }
    }
    if (lane == 31) {
        sh[w] = inc.b;
        sh[16 + w] = inc.o0;
        sh[32 + w] = inc.o1;
    }
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            int x = lane < kWlThreads / 32 ? sh[16 * k + lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int n = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += n;
            }
            if (lane < kWlThreads / 32) sh[16 * k + lane] = x;
        }
    }
    __syncthreads();
    Seg3 ex;
    ex.b = inc.b - v.b + (w ? sh[w - 1] : 0);
    ex.o0 = inc.o0 - v.o0 + (w ? sh[16 + w - 1] : 0);
    ex.o1 = inc.o1 - v.o1 + (w ? sh[32 + w - 1] : 0);
    tot_out->b = sh[kWlThreads / 32 - 1];
    tot_out->o0 = sh[16 + kWlThreads / 32 - 1];
    tot_out->o1 = sh[32 + kWlThreads / 32 - 1];
    __syncthreads();
    return ex;
}

__global__ void __launch_bounds__(kWlThreads) worklist_kernel(const int64_t* __restrict__ offsets,
                                                              const int32_t* __restrict__ indices,
                                                              uint32_t* __restrict__ wl, int32_t* __restrict__ wl_len,
                                                              int64_t BH, int64_t Np, int64_t n_it, int64_t N,
                                                              int32_t pq, int32_t stripe_words, int64_t cap) {
    extern __shared__ uint32_t bm[];  // [4][stripe_words]
    __shared__ int sh[48];
    const int64_t item = blockIdx.x;
    if (offsets[BH * Np] > cap) {  // plan capacity (the CSR's nnz) exceeded: no writes
        if (threadIdx.x == 0) wl_len[3 * item] = wl_len[3 * item + 1] = wl_len[3 * item + 2] = 0;
        return;
    }
    const int64_t bh = item / n_it, it = item % n_it;
    const int G = 256 / pq;
    const int64_t i0 = it * G;
    const int nb = (int)min((int64_t)G, Np - i0);
    const int64_t r0 = bh * Np + i0;
    const int64_t out_base = offsets[r0];
    const int tid = threadIdx.x;
    const int stripe = stripe_words * 32;
    const int n_stripes = (int)((N + stripe - 1) / stripe);
    // tile 0 = blocks [0, G/2), tile 1 = blocks [G/2, G)
    const uint32_t t0mask = G == 4 ? 0x3u : 0x1u;
    Seg3 total = {0, 0, 0};   // segment lengths (pass 0 counts them when striped)
    Seg3 run = {0, 0, 0};     // running output position per segment
    for (int pass = (n_stripes > 1 ? 0 : 1); pass < 2; ++pass) {
        run = {0, 0, 0};
        for (int64_t ss = 0; ss < N; ss += stripe) {
            const int words = (int)min((int64_t)stripe_words, (N - ss + 31) / 32);
            for (int x = tid; x < 4 * stripe_words; x += kWlThreads) bm[x] = 0u;
            __syncthreads();
            // Lists are sorted, so keys sharing a bitmap word sit in adjacent lanes: OR them
            // within the warp (segmented by word) and issue one atomicOr per distinct word.
            for (int b = 0; b < nb; ++b) {
                const int64_t a = offsets[r0 + b], e = offsets[r0 + b + 1];
                constexpr int U = 8;  // independent loads in flight per thread
                for (int64_t tb = a; tb < e; tb += (int64_t)kWlThreads * U) {
                  int32_t kv[U];
#pragma unroll
                  for (int u = 0; u < U; ++u) {
                      const int64_t t = tb + (int64_t)u * kWlThreads + tid;
                      kv[u] = t < e ? __ldg(indices + t) : -1;
                  }
#pragma unroll
                  for (int u = 0; u < U; ++u) {
                    const int64_t key = kv[u];
                    const bool in = key >= ss && key < ss + stripe;
                    const int kk = in ? (int)(key - ss) : 0;
                    const int word = in ? (kk >> 5) : -1 - (tid & 31);  // unique dummy per lane
                    uint32_t bits = in ? (1u << (kk & 31)) : 0u;
                    const int lane = tid & 31;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {  // suffix-OR over lanes with the same word
                        const uint32_t ob = __shfl_down_sync(0xffffffffu, bits, o);
                        const int ow = __shfl_down_sync(0xffffffffu, word, o);
                        if (lane + o < 32 && ow == word) bits |= ob;
                    }
                    const int pw = __shfl_up_sync(0xffffffffu, word, 1);
                    const bool head = lane == 0 || pw != word;
                    if (in && head) atomicOr(&bm[b * stripe_words + word], bits);
                  }
                }
            }
            __syncthreads();
            const int per = (words + kWlThreads - 1) / kWlThreads;
            const int w0 = min(words, tid * per), w1 = min(words, w0 + per);
            Seg3 cnt = {0, 0, 0};
            for (int x = w0; x < w1; ++x) {
                const uint32_t b0 = bm[x], b1 = bm[stripe_words + x], b2 = bm[2 * stripe_words + x],
                               b3 = bm[3 * stripe_words + x];
                const uint32_t u0 = t0mask == 0x3u ? (b0 | b1) : b0;
                const uint32_t u1 = t0mask == 0x3u ? (b2 | b3) : b1;
                cnt.b += __popc(u0 & u1);
                cnt.o0 += __popc(u0 & ~u1);
                cnt.o1 += __popc(u1 & ~u0);
            }
            Seg3 stot;
            const Seg3 ex = block_scan3(cnt, &stot, sh);
            if (pass == 1) {
                const Seg3 seg_base = n_stripes > 1 ? total : stot;  // full segment lengths
                int64_t pb = out_base + run.b + ex.b;
                int64_t p0 = out_base + seg_base.b + run.o0 + ex.o0;
                int64_t p1 = out_base + seg_base.b + seg_base.o0 + run.o1 + ex.o1;
                for (int x = w0; x < w1; ++x) {
                    const uint32_t b0 = bm[x], b1 = bm[stripe_words + x], b2 = bm[2 * stripe_words + x],
                                   b3 = bm[3 * stripe_words + x];
                    const uint32_t u0 = t0mask == 0x3u ? (b0 | b1) : b0;
                    const uint32_t u1 = t0mask == 0x3u ? (b2 | b3) : b1;
                    uint32_t u = u0 | u1;
                    while (u) {
                        const int bit = __ffs(u) - 1;
                        const uint32_t m = 1u << bit;
                        const uint32_t mem = ((b0 & m) ? 1u : 0u) | ((b1 & m) ? 2u : 0u) | ((b2 & m) ? 4u : 0u) |
                                             ((b3 & m) ? 8u : 0u);
                        const uint32_t e = (uint32_t)(ss + x * 32 + bit) | (mem << 28);
                        if ((u0 & m) && (u1 & m)) wl[pb++] = e;
                        else if (u0 & m) wl[p0++] = e;
                        else wl[p1++] = e;
                        u &= u - 1;
                    }
                }
                if (n_stripes == 1) total = stot;
            }
            run.b += stot.b;
            run.o0 += stot.o0;
            run.o1 += stot.o1;
            __syncthreads();
        }
        if (pass == 0) total = run;
    }
    if (tid == 0) {
        wl_len[3 * item] = total.b;
        wl_len[3 * item + 1] = total.o0;
        wl_len[3 * item + 2] = total.o1;
    }
}

cudaError_t launch_worklist(const int64_t* offsets, const int32_t* indices, uint32_t* wl, int32_t* wl_len,
                            int64_t BH, int64_t Np, int64_t n_it, int64_t N, int32_t pq, int64_t cap,
                            cudaStream_t st) {
    const int64_t items = BH * n_it;
    if (items <= 0) return cudaSuccess;
    const int stripe_words = (int)min((int64_t)kStripeWords, (N + 31) / 32);
    const int smem = 4 * stripe_words * 4;
    cudaError_t e = cudaFuncSetAttribute(worklist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    worklist_kernel<<<(unsigned)items, kWlThreads, smem, st>>>(offsets, indices, wl, wl_len, BH, Np, n_it, N, pq,
                                                               stripe_words, cap);
    return cudaGetLastError();
}

template <int D, bool GATHER>
static cudaError_t launch_attn_t(const AttnParams& p, int grid, cudaStream_t st) {
    using C = AttnCfg<D>;
    auto kern = attn_kernel<D, GATHER>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, C::kSmem, st>>>(p);
    return cudaGetLastError();
}

bool attn_uses_pair(const AttnParams& p, int D, bool gather) {
    // The CTA-pair kernel is correct but slower than the double-buffered single-SM kernel on
    // the dit128k plan (84 vs 74 ms, profiles/ubench_r02.md): opt-in with VECATTN_PAIR=1.
    if (!gather || p.causal || D != 128 || p.rep_n > 0 || p.o_mc != nullptr || p.total_items != p.BH * p.n_mt)
        return false;
    const char* e = getenv("VECATTN_PAIR");
    return e != nullptr && e[0] == '1';
}

cudaError_t launch_attn(const AttnParams& p, int D, bool gather, int grid, cudaStream_t st) {
    // Non-causal sparse plans are dominated by chunks of one tile (segments tile 0 / tile 1
    // only), where the double-buffered 64-key kernel (attn_db.cu) is faster; the 128-key
    // ping-pong kernel wins for dense and causal (profiles/sweep_r01.md vs sweep_r01v6.md).
    if (gather && !p.causal) {
        // D = 128 with VECATTN_PAIR=1: the CTA-pair kernel (attn_pair.cu); otherwise the
        // single-SM double-buffered kernel (attn_db.cu).
        if (attn_uses_pair(p, D, gather)) return launch_attn_pair(p, attn_pair_grid(p.total_items, grid_sms()), st);
        return launch_attn_db(p, D, grid, st);
    }
    if (D == 128) return gather ? launch_attn_t<128, true>(p, grid, st) : launch_attn_t<128, false>(p, grid, st);
    if (D == 64) return gather ? launch_attn_t<64, true>(p, grid, st) : launch_attn_t<64, false>(p, grid, st);
    return cudaErrorInvalidValue;
}

}  // namespace va
