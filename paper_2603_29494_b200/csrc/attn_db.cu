// attn_db.cu — vector-sparse attention (Eq. 5, Alg. 2), non-causal variant with a
// DOUBLE-BUFFERED S per tile and 64-key chunks (sm_100a).  launch_attn (attn.cu) uses it
// for the non-causal gather path, where the sparse plan has many single-tile chunks and
// per-tile double buffering beats the 128-key single-buffered ping-pong of attn.cu
// (profiles/sweep_r01.md vs sweep_r01v6.md).
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
//  * 64-key chunks, 4-stage K and V rings; K/V rows gathered with TMA tile::gather4
//    (4 rows x 128 B per instruction) by 2 K-loader and 2 V-loader warps (32 keys
//    each, plan entries prefetched one chunk ahead); dense mode uses 64x64 TMA tiles.
//  * MMA warp: S_t = Q_t K^T (M=128, N=64) into double-buffered TMEM per tile, issued
//    one chunk ahead; O_t += P_t V with A = P_t from TMEM (bf16, written by the softmax
//    over S_t) and B = V (MN-major) from shared memory.
//  * Softmax warpgroup t (thread = query row = TMEM lane): row max in a first TMEM
//    pass, lazy rescale (threshold 2^8, warp-voted because tcgen05.ld/st are
//    warp-collective), exp2 with f32x2 FMA/ADD in a second pass.
//  * Persistent CTAs, dynamic atomic scheduler, items head-major (one head's K/V
//    stays L2-resident), causal items longest-first.
// Degenerate rows (no visible selected key; reading R6): O_r = V_r,
// LSE_r = scale*<q_r,k_r>.
#include "common.cuh"
#include "kernels.cuh"
#include "attn_plan.cuh"

#include <math.h>

namespace va {
namespace db {

namespace {

// VA_DB_WARP_WAIT (build knob): loader warps wait on their EMPTY barriers with every lane
// (1) or with lane 0 behind a divergent branch (0).
#ifndef VA_DB_WARP_WAIT
#define VA_DB_WARP_WAIT 1
#endif
constexpr int kThreads = 448;  // w0 sched+Q, w1 MMA, w2-5 softmax tile 0, w6-9 softmax tile 1, w10-13 loaders
constexpr int kLoadWarps = 4;
constexpr int kFirstLoadWarp = 10;
constexpr int kSoftmaxThreads = 256;
constexpr int kChunk = 64;                  // keys per K/V chunk
constexpr uint32_t kKeyMask = 0x0FFFFFFFu;  // entry = key | membership << 28
constexpr uint32_t kPad = 0x0FFFFFFFu;      // meta key for padding lanes (sorts last)

template <int D>
struct AttnCfg {
    static constexpr int kStages = D == 128 ? 4 : 8;   // K ring (and Q_ext/K_ext bias rows)
#ifndef VA_DB_VSTAGES
#define VA_DB_VSTAGES 4
#endif
    // V ring depth (build knob): a chunk's V gathers are issued after its K gathers and its
    // stage frees only when PV(c - VS) completes, so V lands just in time for PV (%globaltimer
    // trace: PV waits ~0.8 us per chunk on V).  VS = 5 fits in shared memory but is slower in
    // the full step (attention 76.8 vs 74.4 ms, A/B in one box run): the remaining L1 shrinks,
    // and the side-stream CSR emission no longer fits beside the attention CTA.
    static constexpr int kVStages = D == 128 ? VA_DB_VSTAGES : 8;
    static constexpr int kCB = D / 64;
    static constexpr int kQTileBytes = kCB * 128 * 128;   // 128 rows x D bf16
    static constexpr int kKVBytes = kCB * kChunk * 128;    // 64 keys x D bf16
    static constexpr int kOffQ = 0;                        // two Q tiles
    static constexpr int kOffK = 2 * kQTileBytes;
    static constexpr int kOffV = kOffK + kStages * kKVBytes;
    static constexpr int kOffMeta = kOffV + kVStages * kKVBytes;
    static constexpr int kOffQx = (kOffMeta + kVStages * kChunk * 4 + 1023) / 1024 * 1024;  // Q_ext [2][128 x 16]
    static constexpr int kOffKx = kOffQx + 2 * 128 * 16 * 2;                               // K_ext [S][64 x 16]
    static constexpr int kOffBar = kOffKx + kStages * kChunk * 16 * 2;
    static constexpr int B_QFULL = 0, B_QEMPTY = 1, B_KFULL = 2, B_KEMPTY = B_KFULL + kStages,
                         B_VFULL = B_KEMPTY + kStages, B_VEMPTY = B_VFULL + kVStages,
                         B_MFULL = B_VEMPTY + kVStages, B_SFULL = B_MFULL + kVStages /* [2 tiles][2 bufs] */,
                         B_PFULL = B_SFULL + 4, B_ODONE = B_PFULL + 4, B_OEMPTY = B_ODONE + 2,
                         B_IFULL = B_OEMPTY + 2, B_IEMPTY = B_IFULL + 2, B_OFIN = B_IEMPTY + 2, kNumBars = B_OFIN + 2;
    static constexpr int kOffItem = kOffBar + kNumBars * 8;
    static constexpr int kSmem = kOffItem + 16;
    static_assert(kSmem <= 227 * 1024, "shared memory");
    // TMEM: O_t at 128t (D cols); S[t][b] at 256 + 128t + 64b (64 cols; P over its first 32)
    static constexpr uint32_t kTmemCols = 512;
    static constexpr uint32_t kIdescS = make_idesc_bf16(128, kChunk, 0, 0);
    static constexpr uint32_t kIdescPV = make_idesc_bf16(128, D, 0, 1);
};

VA_DEV uint32_t s_col(int t, int b) { return 256u + 128u * t + 64u * b; }

using plan::Chunk;
using plan::Item;
using plan::trace;
template <bool G>
VA_DEV Item decode_item(const AttnParams& p, int item) { return plan::decode_item<kChunk, G>(p, item); }
template <bool G>
VA_DEV Chunk chunk_info(const Item& I, int j) { return plan::chunk_info<kChunk, G>(I, j); }

VA_DEV uint32_t prefix_mask(int64_t nb) { return nb >= 32 ? 0xffffffffu : (nb <= 0 ? 0u : ((1u << nb) - 1u)); }

}  // namespace

template <int D, bool GATHER>
__global__ void __launch_bounds__(kThreads, 1) attn_db_kernel(const __grid_constant__ AttnParams p) {
    using C = AttnCfg<D>;
    constexpr int S_ = C::kStages;
    constexpr int VS = C::kVStages;
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
            mbar_init(&bars[C::B_KFULL + s], 1);
            mbar_init(&bars[C::B_KEMPTY + s], 1);
        }
        for (int s = 0; s < VS; ++s) {
            mbar_init(&bars[C::B_VFULL + s], 1);
            mbar_init(&bars[C::B_VEMPTY + s], 1);
            mbar_init(&bars[C::B_MFULL + s], 1);
        }
        for (int x = 0; x < 4; ++x) {
            mbar_init(&bars[C::B_SFULL + x], 1);
            mbar_init(&bars[C::B_PFULL + x], 128);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&bars[C::B_ODONE + t], 1);
            mbar_init(&bars[C::B_OEMPTY + t], 128);
            mbar_init(&bars[C::B_IFULL + t], 1);
            mbar_init(&bars[C::B_IEMPTY + t], 1 + kSoftmaxThreads + kLoadWarps);
            mbar_init(&bars[C::B_OFIN + t], 1);
        }
        fence_barrier_init();
    }
    if constexpr (GATHER) {
        // Membership masking on the tensor core: S = [Q | E] [K | F]^T with E = one-hot of the
        // row's block (Q_ext, constant per row position) and F[j][b] = 0 if key j is in block
        // b's index set else -2^100 (K_ext, written per chunk by the K loaders).  Members get
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
                if (qi > 0) mbar_wait_long(&bars[C::B_QEMPTY], (qi - 1) & 1);  // waits out an item
                mbar_arrive_expect_tx(&bars[C::B_QFULL], 2 * C::kQTileBytes);
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int cb = 0; cb < C::kCB; ++cb)
                        tma_load_3d_hint(sQ + t * C::kQTileBytes + cb * 128 * 128, &p.tm_q, &bars[C::B_QFULL],
                                         cb * 64, (int)(I.it * 256 + t * 128), (int)I.bh, pol_stream);
            }
            ++qi;
        }
    } else if (warp >= kFirstLoadWarp) {
        // ======================================== K/V loaders (4 warps)
        // Warp g owns every chunk c = g (mod 4): K and V of all 64 keys.  A warp's TMA issue
        // rate is bound by a fixed per-iteration cost plus ~70 clk per gather4 (uniform-register
        // setup), so whole chunks per warp (fewer iterations each) beat splitting every chunk
        // across warps (scripts/ubench_gather.cu).  Stage s = c % S_ with S_ % 4 == 0, so the
        // previous chunk on a stage is this warp's own and its EMPTY parity waits are exact.
        // GATHER: two plan entries per lane (keys lane, 32+lane; prefetched one owned chunk
        // ahead), lanes 0-15 issue the tile::gather4s; K_ext bias rows are written before the
        // K gathers (consumed by the S MMA, freed with KEMPTY), the keys for the causal mask
        // before the V gathers (freed with VEMPTY).
        // VA_DB_KV_SPLIT: warps 0-1 load only K (chunks c = g mod 2), warps 2-3 only V, so a
        // chunk's V gathers do not queue behind its K gathers in one warp.
#ifndef VA_DB_KV_SPLIT
#define VA_DB_KV_SPLIT 0
#endif
        constexpr bool kSplit = VA_DB_KV_SPLIT != 0;
        constexpr int NW = kSplit ? kLoadWarps / 2 : kLoadWarps;  // warps per role
        static_assert(S_ % NW == 0, "stage ownership");
        const int g0 = (int)warp - kFirstLoadWarp;
        const bool k_role = !kSplit || g0 < NW, v_role = !kSplit || g0 >= NW;
        const int g = kSplit ? g0 % NW : g0;
        int64_t c = 0;  // chunks of all previous items
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
            int j = (int)(((int64_t)g - c % NW + NW) % NW);  // first owned chunk
            if constexpr (GATHER) {
                const uint32_t* wlp = p.wl + I.base;
                Chunk ch;
                ch.len = 0;
                ch.start = 0;
                if (j < I.n_chunks) ch = chunk_info<true>(I, j);
                uint32_t e0 = (int)lane < ch.len ? __ldcs(wlp + ch.start + lane) : 0u;
                uint32_t e1 = 32 + (int)lane < ch.len ? __ldcs(wlp + ch.start + 32 + lane) : 0u;
                for (; j < I.n_chunks; j += NW) {
                    const int64_t cc = c + j;
                    const int s = (int)(cc % S_);
                    const int round = (int)(cc / S_);
                    Chunk chn;
                    chn.len = 0;
                    chn.start = 0;
                    if (j + NW < I.n_chunks) chn = chunk_info<true>(I, j + NW);
                    const uint32_t en0 = (int)lane < chn.len ? __ldcs(wlp + chn.start + lane) : 0u;
                    const uint32_t en1 = 32 + (int)lane < chn.len ? __ldcs(wlp + chn.start + 32 + lane) : 0u;
                    const bool ok0 = (int)lane < ch.len, ok1 = 32 + (int)lane < ch.len;
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
                    if (k_role) {
#if VA_DB_WARP_WAIT
                    if (round > 0) mbar_wait(&bars[C::B_KEMPTY + s], (round - 1) & 1);  // all lanes: no divergence
#else
                    if (lane == 0 && round > 0) mbar_wait(&bars[C::B_KEMPTY + s], (round - 1) & 1);
#endif
                    if (lane == 0) trace(p, 0, cc);
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
                        *reinterpret_cast<uint4*>(kx + k16_offset((int)lane, 0)) = bias(m0);
                        *reinterpret_cast<uint4*>(kx + k16_offset(32 + (int)lane, 0)) = bias(m1);
                        fence_proxy_async();  // generic-proxy smem write -> tcgen05.mma (async proxy)
                    }
                    __syncwarp();
                    mbar_arrive_expect_tx_if(&bars[C::B_KFULL + s], kChunk * D * 2, lane == 0);
                    if (lane < 16) {
                        uint8_t* dst = sK + s * C::kKVBytes + 4 * (int)lane * 128;
#pragma unroll
                        for (int cb = 0; cb < C::kCB; ++cb)
                            tma_gather4(dst + cb * kChunk * 128, &p.tm_k, &bars[C::B_KFULL + s], cb * 64, ra, rb, rc,
                                        rd);
                    }
                    }
                    // ---- V: keys for the causal mask, then the gathers.  V stage sv = cc % VS
                    // is not owned by one warp (VS % 4 != 0), but the wait stays unambiguous:
                    // this warp's previous V wait (chunk cc - 4) proved PV(cc - 4 - VS) done, so
                    // PV(cc - 2 VS) -- the phase before the one waited for -- is complete.
                    if (v_role) {
                    const int sv = (int)(cc % VS), vround = (int)(cc / VS);
#if VA_DB_WARP_WAIT
                    if (vround > 0) mbar_wait(&bars[C::B_VEMPTY + sv], (vround - 1) & 1);
#else
                    if (lane == 0 && vround > 0) mbar_wait(&bars[C::B_VEMPTY + sv], (vround - 1) & 1);
#endif
                    if (lane == 0) trace(p, 1, cc);
                    __syncwarp();  // every lane after lane 0's VEMPTY wait (the V gathers below)
                    if (p.causal) {  // the causal softmax's per-row prefix search reads the keys
                        sMeta[sv * kChunk + lane] = ok0 ? key0 : kPad;
                        sMeta[sv * kChunk + 32 + lane] = ok1 ? key1 : kPad;
                        __syncwarp();
                    }
                    // the causal-key hand-off has a waiter only in the causal softmax (an
                    // unobserved arrive is what compute-sanitizer synccheck flags)
                    mbar_arrive_if(&bars[C::B_MFULL + sv], lane == 0 && p.causal);
                    mbar_arrive_expect_tx_if(&bars[C::B_VFULL + sv], kChunk * D * 2, lane == 0);
                    if (lane < 16) {
                        uint8_t* dst = sV + sv * C::kKVBytes + 4 * (int)lane * 128;
#pragma unroll
                        for (int cb = 0; cb < C::kCB; ++cb)
                            tma_gather4(dst + cb * kChunk * 128, &p.tm_v, &bars[C::B_VFULL + sv], cb * 64, ra, rb, rc,
                                        rd);
                    }
                    }
                    e0 = en0;
                    e1 = en1;
                    ch = chn;
                }
            } else {
                if (lane == 0 && !kSplit) {
                    for (; j < I.n_chunks; j += kLoadWarps) {
                        const int64_t cc = c + j;
                        const int s = (int)(cc % S_);
                        const int round = (int)(cc / S_);
                        if (round > 0) mbar_wait(&bars[C::B_KEMPTY + s], (round - 1) & 1);
                        mbar_arrive_expect_tx(&bars[C::B_KFULL + s], C::kKVBytes);
#pragma unroll
                        for (int cb = 0; cb < C::kCB; ++cb)
                            tma_load_3d(sK + s * C::kKVBytes + cb * kChunk * 128, &p.tm_k, &bars[C::B_KFULL + s],
                                        cb * 64, j * kChunk, (int)bh_kv);
                        const int sv = (int)(cc % VS), vround = (int)(cc / VS);
                        if (vround > 0) mbar_wait(&bars[C::B_VEMPTY + sv], (vround - 1) & 1);
                        mbar_arrive_expect_tx(&bars[C::B_VFULL + sv], C::kKVBytes);
#pragma unroll
                        for (int cb = 0; cb < C::kCB; ++cb)
                            tma_load_3d(sV + sv * C::kKVBytes + cb * kChunk * 128, &p.tm_v, &bars[C::B_VFULL + sv],
                                        cb * 64, j * kChunk, (int)bh_kv);
                    }
                }
                __syncwarp();
            }
            c += I.n_chunks;
        }
    } else if (warp == 1) {
        // ======================================== MMA issuer (single thread)
        // Per chunk c: S_t(c+1) for the tiles of chunk c+1 (double-buffered S, so it can run
        // ahead of the softmax of c), then PV_t(c) for the tiles of chunk c.
        if (elect_one()) {
            int64_t c = 0;                 // global chunk counter (stage rings)
            uint32_t ns[2] = {0, 0};       // S issued per tile (buffer = ns & 1)
            uint32_t np_[2] = {0, 0};      // PV issued per tile
            int qi = 0, oi = 0;
            const uint32_t qa = smem_u32(sQ);
            auto wait_k = [&](int64_t cc) {
                mbar_wait(&bars[C::B_KFULL + (int)(cc % S_)], (uint32_t)((cc / S_) & 1));
                tc_fence_after();
                trace(p, 2, cc);
            };
            auto issue_s = [&](int t, int64_t cc) {
                const int s = (int)(cc % S_);
                const int bi = (int)(ns[t] & 1u);
                const uint32_t ka = smem_u32(sK + s * C::kKVBytes);
                const uint32_t q_t = qa + t * C::kQTileBytes;
                const uint32_t st = tmem_base + s_col(t, bi);
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
                mma_commit(&bars[C::B_SFULL + 2 * t + bi]);
                ++ns[t];
            };
            auto issue_pv = [&](int t, int64_t cc, bool first) {
                const int s = (int)(cc % VS);
                const int bi = (int)(np_[t] & 1u);
                mbar_wait(&bars[C::B_PFULL + 2 * t + bi], (np_[t] >> 1) & 1u);
                ++np_[t];
                tc_fence_after();
                const uint32_t pt = tmem_base + s_col(t, bi);
                const uint32_t ot = tmem_base + 128u * t;
                const uint32_t va = smem_u32(sV + s * C::kKVBytes);
#pragma unroll
                for (int kk = 0; kk < kChunk / 16; ++kk) {
                    const uint64_t bdesc = make_sdesc(va + kk * 16 * 128, kChunk * 128, 1024);
                    mma_bf16_ts(ot, pt + kk * 8, bdesc, C::kIdescPV, (first && kk == 0) ? 0u : 1u);
                }
                mma_commit(&bars[C::B_ODONE + t]);
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
                if (oi > 0) {  // O_0 / O_1 of the previous item drained by the epilogues
                    mbar_wait(&bars[C::B_OEMPTY + 0], (oi - 1) & 1);
                    mbar_wait(&bars[C::B_OEMPTY + 1], (oi - 1) & 1);
                }
                ++oi;
                bool started[2] = {false, false};
                int m = chunk_info<GATHER>(I, 0).mask;
                wait_k(c);
                if (m & 1) issue_s(0, c);
                if (m & 2) issue_s(1, c);
                mma_commit(&bars[C::B_KEMPTY + (int)(c % S_)]);
                if (I.n_chunks == 1) mma_commit(&bars[C::B_QEMPTY]);
                for (int j = 0; j < I.n_chunks; ++j, ++c) {
                    const bool more = j + 1 < I.n_chunks;
                    int mn = 0;
                    auto issue_next_s = [&]() {
                        mn = chunk_info<GATHER>(I, j + 1).mask;
                        if (mn & 1) issue_s(0, c + 1);
                        if (mn & 2) issue_s(1, c + 1);
                        mma_commit(&bars[C::B_KEMPTY + (int)((c + 1) % S_)]);
                        if (j + 2 == I.n_chunks) mma_commit(&bars[C::B_QEMPTY]);
                    };
                    // S(j+1) first if its K chunk has landed (softmax(j+1) can then overlap
                    // PV(j)); otherwise PV(j) first so the tensor core does not idle on the gather
                    bool s_first = false;
                    if (more) {
                        const int64_t cn = c + 1;
                        s_first = mbar_try_wait(&bars[C::B_KFULL + (int)(cn % S_)], (uint32_t)((cn / S_) & 1));
                        if (s_first) {
                            tc_fence_after();
                            trace(p, 2, cn);
                            issue_next_s();
                        }
                    }
                    mbar_wait(&bars[C::B_VFULL + (int)(c % VS)], (uint32_t)((c / VS) & 1));
                    trace(p, 3, c);
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        if (!(m & (1 << t))) continue;
                        issue_pv(t, c, !started[t]);
                        started[t] = true;
                        trace(p, 4 + t, c);
                    }
                    mma_commit(&bars[C::B_VEMPTY + (int)(c % VS)]);
                    if (more && !s_first) {
                        wait_k(c + 1);
                        issue_next_s();
                    }
                    m = mn;
                }
                // O_0 / O_1 final for this item (one phase per item with chunks, both tiles)
                mma_commit(&bars[C::B_OFIN + 0]);
                mma_commit(&bars[C::B_OFIN + 1]);
            }
        }
        __syncwarp();
    } else {
        // ======================================== softmax / epilogue (two warpgroups)
        const int tile = ((int)warp - 2) >> 2;
        const uint32_t quad = warp & 3u;
        const int r = (int)(quad * 32 + lane);
        const uint32_t lane_off = (quad * 32u) << 16;
        const uint32_t tO = tmem_base + lane_off + 128u * tile;
        const int row_in_item = 128 * tile + r;
        const float sl2 = p.scale_log2;
        int64_t c = 0;
        uint32_t ct = 0;  // this tile's chunk counter (S buffer = ct & 1)
        uint32_t od = 0;  // ODONE phases known complete (= PVs of this tile known finished)
        uint32_t fi = 0;  // OFIN phases waited (items with chunks)
        for (int it = 0;; ++it) {
            const int slot = it & 1;
            mbar_wait(&bars[C::B_IFULL + slot], (it >> 1) & 1);
            const int item = item_slot[slot];
            mbar_arrive(&bars[C::B_IEMPTY + slot]);
            if (item < 0) break;
            const Item I = decode_item<GATHER>(p, item);
            const int64_t qrow = I.it * 256 + row_in_item;
            const bool row_ok = qrow < p.N;
            float m_ref = -INFINITY;  // log2-domain reference max (lazy rescaling)
            float2 lsum2 = make_float2(0.f, 0.f);
            // this tile's chunks only: the shared ones, then its own (no per-chunk plan walk over
            // the other tile's chunks); a chunk's position in the item (plan::own_chunk) is needed
            // only for the causal key hand-off, which is indexed by the global chunk counter
            const int n_own = GATHER ? I.nb + (tile == 0 ? I.n0 : I.n1) : I.n_chunks;
            int jt = 0;  // chunks of this item processed by this tile
            for (; jt < n_own;) {
                int64_t cj = c;
                if constexpr (GATHER) {
                    if (p.causal) cj = c + plan::own_chunk(I, tile, jt);
                } else {
                    cj = c + jt;
                }
                const int bi = (int)(ct & 1u);
                const uint32_t tS = tmem_base + lane_off + s_col(tile, bi);
                uint32_t mw[2];
                if constexpr (GATHER) {
                    mw[0] = mw[1] = 0xffffffffu;  // membership is applied by the MMA
                    if (p.causal) {
                        mbar_wait(&bars[C::B_MFULL + (int)(cj % VS)], (uint32_t)((cj / VS) & 1));
                        const uint32_t* meta = sMeta + (int)(cj % VS) * kChunk;
                        int lo = 0, hi = kChunk;  // keys ascending: visible = prefix with key <= qrow
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            if ((int64_t)meta[mid] <= qrow) lo = mid + 1;
                            else hi = mid;
                        }
                        mw[0] = prefix_mask(lo);
                        mw[1] = prefix_mask(lo - 32);
                    }
                } else {
                    const int64_t vend = p.causal ? min(p.N, qrow + 1) : p.N;
                    const int64_t nv = vend - (int64_t)jt * kChunk;
                    mw[0] = prefix_mask(nv);
                    mw[1] = prefix_mask(nv - 32);
                }
                const bool full = (mw[0] & mw[1]) == 0xffffffffu;
                mbar_wait(&bars[C::B_SFULL + 2 * tile + bi], (ct >> 1) & 1u);
                tc_fence_after();
                if (lane == 0 && (warp == 2 || warp == 6)) trace(p, 6 + 2 * tile, cj);
                __syncwarp();  // reconverge after the per-row causal search (tcgen05.ld is .sync.aligned)
                // ---- single TMEM pass (TMEM reads, 64 B/clk/SM, bind at D = 128): S -> registers,
                // masked row max, lazy O rescale, P = exp2(s*scale*log2e - m) bf16-packed over S.
                uint32_t a[32], b[32];
                tmem_ld32(tS, a);
                tmem_ld32(tS + 32, b);
                tmem_ld_wait();
                if (!full) {  // causal / ragged tail only: masked scores -> -inf (exp2 -> 0)
#pragma unroll
                    for (int t = 0; t < 32; ++t) {
                        a[t] = (mw[0] & (1u << t)) ? a[t] : 0xff800000u;
                        b[t] = (mw[1] & (1u << t)) ? b[t] : 0xff800000u;
                    }
                }
                float mx;
                {  // 4 independent FMNMX3 chains (latency), then combine
                    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                    for (int t = 0; t < 32; t += 4) {
                        m4[0] = fmaxf(fmaxf(m4[0], __uint_as_float(a[t])), __uint_as_float(a[t + 1]));
                        m4[1] = fmaxf(fmaxf(m4[1], __uint_as_float(a[t + 2])), __uint_as_float(a[t + 3]));
                        m4[2] = fmaxf(fmaxf(m4[2], __uint_as_float(b[t])), __uint_as_float(b[t + 1]));
                        m4[3] = fmaxf(fmaxf(m4[3], __uint_as_float(b[t + 2])), __uint_as_float(b[t + 3]));
                    }
                    mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
                }
                const float m_new = fmaxf(m_ref, mx * sl2);
                // SFULL(ct) fired, so every MMA issued before S(ct) -- including PV(ct-2) of
                // this tile -- is complete: ODONE phases 0..ct-2 are done (parity waits on
                // phase ct-1 are then unambiguous).
                // Default: the phases are only counted (od), never waited on unless a rescale needs
                // PV(ct-1).  p.strict_sync (VECATTN_STRICT_SYNC=1): every ODONE phase is waited on
                // before the next commit can arrive, which compute-sanitizer synccheck requires (it
                // reports an unobserved mbarrier phase as "missing wait"); ~2% slower at dit128k.
                if (p.strict_sync) {
                    for (; od + 1 < ct; ++od) mbar_wait(&bars[C::B_ODONE + tile], od & 1u);
                } else if (ct >= 1 && od < ct - 1) {
                    od = ct - 1;
                }
                const bool need = m_new > m_ref + 8.0f;
                const float corr = need ? ex2(m_ref - m_new) : 1.0f;
                if (need) {
                    lsum2.x *= corr;
                    lsum2.y *= corr;
                    m_ref = m_new;
                }
                if (jt > 0 && __any_sync(0xffffffffu, need)) {
                    // O_t must be stable (PV_t of this tile's previous chunk done) before the
                    // rescale; without a rescale the softmax never waits on the PV pipeline.
                    for (; od < ct; ++od) mbar_wait(&bars[C::B_ODONE + tile], od & 1u);
                    tc_fence_after();
#pragma unroll
                    for (int g = 0; g < D / 8; ++g) {
                        uint32_t o[8];
                        tmem_ld8(tO + g * 8, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int t = 0; t < 8; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * corr);
                        tmem_st8(tO + g * 8, o);
                    }
                    tmem_st_wait();
                }
                {
                    const float neg_m = (m_ref == -INFINITY) ? 0.f : -m_ref;
                    const uint64_t sl2x2 = pack_f32x2(sl2, sl2);
                    const uint64_t nmx2 = pack_f32x2(neg_m, neg_m);
                    uint32_t pk[32];
#pragma unroll
                    for (int t = 0; t < 32; t += 2) {
                        const float2 xa = unpack_f32x2(
                            ffma2(pack_f32x2(__uint_as_float(a[t]), __uint_as_float(a[t + 1])), sl2x2, nmx2));
                        const float2 xb = unpack_f32x2(
                            ffma2(pack_f32x2(__uint_as_float(b[t]), __uint_as_float(b[t + 1])), sl2x2, nmx2));
                        const float p0 = ex2(xa.x), p1 = ex2(xa.y), p2 = ex2(xb.x), p3 = ex2(xb.y);
                        lsum2 = fadd2(lsum2, fadd2(make_float2(p0, p1), make_float2(p2, p3)));
                        pk[t >> 1] = pack_bf16x2(p0, p1);
                        pk[16 + (t >> 1)] = pack_bf16x2(p2, p3);
                    }
                    tmem_st32(tS, pk);
                    tmem_st_wait();
                }
                if (p.strict_sync)  // PV(ct-1)'s phase, observed before PV(ct) (needs P(ct)) can commit
                    for (; od < ct; ++od) mbar_wait(&bars[C::B_ODONE + tile], od & 1u);
                tc_fence_before();
                mbar_arrive(&bars[C::B_PFULL + 2 * tile + bi]);
                if (lane == 0 && (warp == 2 || warp == 6)) trace(p, 7 + 2 * tile, cj);
                ++ct;
                ++jt;
            }
            c += I.n_chunks;
            // ---------------------------------------------------------------- epilogue
            // rows that only ever saw masked keys carry m_ref ~ -2^100*scale*log2e: no visible key
            const float l = (m_ref < -0x1p99f * sl2) ? 0.f : lsum2.x + lsum2.y;  // scale-aware: masked = -2^100*sl2
            const float inv = l > 0.f ? 1.f / l : 0.f;
            const plan::ORow orow = plan::o_row<D>(p, I.bh, qrow);
            if (I.n_chunks > 0) {  // every PV of the item complete (ODONE parity may be 2 behind here)
                mbar_wait_long(&bars[C::B_OFIN + tile], fi & 1u);
                ++fi;
            }
            if (jt > 0) {
                __syncwarp();
                tc_fence_after();
#pragma unroll
                for (int g = 0; g < D / 32; ++g) {
                    uint32_t ov[32];
                    tmem_ld32(tO + g * 32, ov);
                    tmem_ld_wait();
                    if (row_ok && l > 0.f) {
#pragma unroll
                        for (int t = 0; t < 32; t += 8) {
                            uint4 w;
                            w.x = pack_bf16x2(__uint_as_float(ov[t]) * inv, __uint_as_float(ov[t + 1]) * inv);
                            w.y = pack_bf16x2(__uint_as_float(ov[t + 2]) * inv, __uint_as_float(ov[t + 3]) * inv);
                            w.z = pack_bf16x2(__uint_as_float(ov[t + 4]) * inv, __uint_as_float(ov[t + 5]) * inv);
                            w.w = pack_bf16x2(__uint_as_float(ov[t + 6]) * inv, __uint_as_float(ov[t + 7]) * inv);
                            plan::o_store16<D>(p, orow, g * 32 + t, w);  // streamed: evict first
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


template <int D>
static cudaError_t launch_db_t(const AttnParams& p, int grid, cudaStream_t st) {
    using C = AttnCfg<D>;
    auto kern = attn_db_kernel<D, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, C::kSmem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace db

cudaError_t launch_attn_db(const AttnParams& p, int D, int grid, cudaStream_t st) {
    if (D == 128) return db::launch_db_t<128>(p, grid, st);
    if (D == 64) return db::launch_db_t<64>(p, grid, st);
    return cudaErrorInvalidValue;
}

}  // namespace va
