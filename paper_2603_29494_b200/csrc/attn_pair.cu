// attn_pair.cu — vector-sparse attention (Eq. 5, Alg. 2), non-causal, on a CTA PAIR
// (tcgen05 cta_group::2, cluster of 2 SMs) with 128-key chunks (sm_100a, D = 128).
//
// PAPER.md Eq. 5: for query block i,
//     O[I_B(i)] = softmax( Q[I_B(i)] K[Idx(i)]^T / sqrt(D) ) V[Idx(i)]
// computed with FlashAttention-style online softmax over chunks of gathered K/V rows
// (Alg. 2; App. D.2).
//
// B200 design (DESIGN.md §6 "attn_pair_kernel"):
//  * Work item = 256 query rows (256/P_q adjacent blocks) with the union key plan of
//    attn_plan.cuh (entries key | membership << 28, segments both / tile 0 / tile 1).  The
//    two 128-row tiles of an item live on the two SMs of a cluster: CTA r owns rows
//    [128r, 128r+128), its Q tile, its O accumulator, its softmax.
//  * One leader thread issues M = 256 pair MMAs for both SMs:
//      S  = [Q | E] [K | F]^T   (SS, N = 128 keys: CTA r holds the K rows of chunk keys
//                                [64r, 64r+64) -- half of the B operand; E/F = membership
//                                one-hot / bias, one extra K = 16 step)
//      O += P V                 (TS, A = P from each CTA's TMEM, N = D = 128: CTA r holds
//                                the V columns [64r, 64r+64) of all 128 keys)
//    so each SM gathers 256 B per union key (half of K, half of V) instead of 512 B, and
//    the tensor core runs N = 128 (full rate; scripts/probe_pair.cu: 64 clk per
//    M256 N128 K16 instruction) with half the per-SM shared-memory operand reads.
//  * TMEM per CTA (512 cols): O_0 [0,128), O_1 [128,256), S_0 [256,384), S_1 [384,512).
//    Chunks alternate between two softmax warpgroups (chunk c -> WG c & 1, S_{c&1}, O_{c&1}),
//    FA4-style ping-pong: while WG x exponentiates chunk c the tensor core runs PV(c-1) and
//    S(c+1) for the other WG.  Each WG keeps its own online-softmax state and O accumulator;
//    the two partial results of a row are merged in the epilogue (log-sum-exp weights).
//    A thread holds a whole 128-column S row (setmaxnreg 192 for the softmax warpgroups).
//    A chunk whose keys belong to the other tile only (plan segment) writes P = 0 without
//    the exponentials.
//  * Loaders: kLW chunk-owning warps per CTA; each gathers its CTA's K half (+ bias rows)
//    and V half of the chunk with TMA tile::gather4 and completes on the LEADER's
//    KFULL / VFULL barriers (.cta_group::2), which the MMA thread waits on.
// Degenerate rows (no visible selected key; reading R6): O_r = V_r,
// LSE_r = scale*<q_r,k_r>.
#include "common.cuh"
#include "kernels.cuh"
#include "attn_plan.cuh"

#include <math.h>
#include <algorithm>

namespace va {
namespace pair {

namespace {

constexpr int D = 128;
constexpr int kChunk = 128;                 // keys per chunk (both CTAs)
constexpr int kHalf = 64;                   // K rows per CTA per chunk
constexpr int kStages = 5;                  // K/V ring depth
constexpr int kKW = 4, kVW = 2;             // K-half and V-half loader warps per CTA (w2-3, w12-15)
constexpr int kLW = kKW + kVW;
constexpr int kThreads = (2 + 8 + kLW) * 32;  // w0 sched/Q, w1 MMA, w2-3 loaders, w4-11 softmax, w12-15 loaders
constexpr int kSoftFirst = 4;
#ifndef VA_PAIR_POLY_NUM
#define VA_PAIR_POLY_NUM 0
#endif
#ifndef VA_PAIR_POLY_DEN
#define VA_PAIR_POLY_DEN 4
#endif
constexpr int kPolyNum = VA_PAIR_POLY_NUM, kPolyDen = VA_PAIR_POLY_DEN;  // share of exp2 on the FMA pipe
constexpr uint32_t kKeyMask = 0x0FFFFFFFu;

VA_DEV int loader_index(uint32_t warp) { return warp < 4 ? (int)warp - 2 : (int)warp - 10; }

constexpr int kQBytes = 128 * D * 2;         // 32 KB (2 col blocks x [128 x 64] SW128)
constexpr int kKBytes = kHalf * D * 2;       // 16 KB (2 col blocks x [64 x 64])
constexpr int kVBytes = kChunk * 64 * 2;     // 16 KB ([128 keys x 64 cols] MN-major SW128)
constexpr int kKxBytes = kHalf * 16 * 2;     // 2 KB bias rows
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + kQBytes;
constexpr int kOffV = kOffK + kStages * kKBytes;
constexpr int kOffKx = kOffV + kStages * kVBytes;
constexpr int kOffQx = kOffKx + kStages * kKxBytes;
constexpr int kOffRed = kOffQx + 128 * 16 * 2;   // float [2 WGs][3][128]: epilogue merge (m, l, has)
constexpr int kOffBar = kOffRed + 2 * 3 * 128 * 4;
enum {
    B_IFULL = 0, B_IEMPTY = 2, B_QFULL = 4, B_QEMPTY = 5, B_KFULL = 6, B_KEMPTY = B_KFULL + kStages,
    B_VFULL = B_KEMPTY + kStages, B_VEMPTY = B_VFULL + kStages, B_SFULL = B_VEMPTY + kStages,
    B_PFULL = B_SFULL + 2, B_OFIN = B_PFULL + 2, B_OEMPTY = B_OFIN + 1,
    B_DONE = B_OEMPTY + 1, kNumBars = B_DONE + 1
};
constexpr int kOffItem = kOffBar + kNumBars * 8;
constexpr int kSmem = kOffItem + 16;
static_assert(kSmem <= 227 * 1024, "smem");

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kIdescS = make_idesc_bf16(256, kChunk, 0, 0);
constexpr uint32_t kIdescPV = make_idesc_bf16(256, D, 0, 1);
VA_DEV uint32_t o_col(int x) { return 128u * (uint32_t)x; }
VA_DEV uint32_t s_col(int x) { return 256u + 128u * (uint32_t)x; }
VA_DEV void setmaxnreg_inc192() { asm volatile("setmaxnreg.inc.sync.aligned.u32 192;"); }
VA_DEV void setmaxnreg_dec64() { asm volatile("setmaxnreg.dec.sync.aligned.u32 64;"); }
// consumers of an item slot: leader {MMA, loaders, softmax}, peer {Q loader, loaders, softmax}
constexpr int kSlotConsumers = 2 * (1 + kLW + 8);

using plan::Chunk;
using plan::Item;
VA_DEV Item decode(const AttnParams& p, int item) { return plan::decode_item<kChunk, true>(p, item); }
VA_DEV Chunk chunk(const Item& I, int j) { return plan::chunk_info<kChunk, true>(I, j); }

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_pair_kernel(const __grid_constant__ AttnParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sQ = smem + kOffQ;
    uint8_t* sK = smem + kOffK;
    uint8_t* sV = smem + kOffV;
    float* sRed = reinterpret_cast<float*>(smem + kOffRed);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
    int* item_slot = reinterpret_cast<int*>(smem + kOffItem);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffItem + 8);

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    // capacity protocol of the fused path: both CTAs see the same value, so both return
    if (p.d_nnz != nullptr && *p.d_nnz > p.nnz_cap) return;

    if (threadIdx.x == 0) {
        if ((smem_u32(smem) & 1023u) != 0) __trap();
        for (int x = 0; x < 2; ++x) {
            mbar_init(&bars[B_IFULL + x], 1);
            mbar_init(&bars[B_IEMPTY + x], kSlotConsumers);
        }
        mbar_init(&bars[B_QFULL], 1);
        mbar_init(&bars[B_QEMPTY], 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars[B_KFULL + s], 2 * kKW);  // K warps of both CTAs (bias rows written; leader's warp 0 expect_tx)
            mbar_init(&bars[B_KEMPTY + s], 1);
            mbar_init(&bars[B_VFULL + s], 1);  // leader loader (expect_tx); the peer's bytes complete_tx
            mbar_init(&bars[B_VEMPTY + s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bars[B_SFULL + b], 1);
            mbar_init(&bars[B_PFULL + b], 8);  // the WG's 4 softmax warps x 2 CTAs
        }
        mbar_init(&bars[B_OFIN], 1);
        mbar_init(&bars[B_OEMPTY], 16);
        mbar_init(&bars[B_DONE], 8);  // this CTA's softmax warps have finished
        fence_barrier_init();
    }
    {
        // Membership masking on the tensor core (as attn_db.cu): E = one-hot of the row's block
        // within the item, F[j][b] = 0 if key j is in block b's set else -2^100 (written per
        // chunk by the loaders for this CTA's K half).
        uint16_t* qx = reinterpret_cast<uint16_t*>(smem + kOffQx);
        for (int x = threadIdx.x; x < 128 * 16; x += kThreads) {
            const int r = x / 16, e = x % 16;
            const int blk = (128 * (int)rank + r) / p.pq;
            qx[k16_offset(r, e) / 2] = (e == blk) ? 0x3F80u : 0u;  // bf16 1.0
        }
        uint32_t* kx = reinterpret_cast<uint32_t*>(smem + kOffKx);
        for (int x = threadIdx.x; x < kStages * kKxBytes / 4; x += kThreads) kx[x] = 0u;
        fence_proxy_async();
    }
    if (warp == 1) tmem_alloc_pair<kTmemCols>(tmem_slot);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // leader-CTA barrier addresses (shared::cluster) for the peer's remote arrivals / TMA completion
    auto lbar = [&](int i) { return mapa_rank(smem_u32(&bars[i]), 0); };
    auto arrive_leader = [&](int i) {
        if (leader) mbar_arrive(&bars[i]);
        else mbar_arrive_cluster_relaxed(lbar(i));  // item slot consumed: the value is in a register
    };

    const bool softmax_wg = warp >= (uint32_t)kSoftFirst && warp < (uint32_t)kSoftFirst + 8;
    if (!softmax_wg) {
    setmaxnreg_dec64();  // whole warpgroups WG0 / WG3 (setmaxnreg is warpgroup-collective)
    if (warp == 0) {
        // ============================== leader: scheduler + Q; peer: Q loader
        if (lane == 0) {
            tma_prefetch_desc(&p.tm_q);
            tma_prefetch_desc(&p.tm_k);
            tma_prefetch_desc(&p.tm_v);
        }
        const uint64_t pol_stream = l2_evict_first_policy();
        const uint32_t qfull_l = lbar(B_QFULL);
        int qi = 0;
        for (int it = 0;; ++it) {
            const int slot = it & 1;
            int item = 0;
            if (leader) {
                if (lane == 0) {
                    if (it >= 2) mbar_wait_cl(&bars[B_IEMPTY + slot], ((it >> 1) - 1) & 1);
                    item = atomicAdd(p.work_counter, 1);
                    if (item >= p.total_items) item = -1;
                    item_slot[slot] = item;
                    st_cluster_u32(mapa_rank(smem_u32(&item_slot[slot]), 1), (uint32_t)item);
                    mbar_arrive(&bars[B_IFULL + slot]);
                    mbar_arrive_cluster(mapa_rank(smem_u32(&bars[B_IFULL + slot]), 1));
                }
                item = __shfl_sync(0xffffffffu, item, 0);
            } else {
                mbar_wait_cl(&bars[B_IFULL + slot], (it >> 1) & 1);
                item = item_slot[slot];
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster_relaxed(lbar(B_IEMPTY + slot));
            }
            if (item < 0) break;
            const Item I = decode(p, item);
            if (I.n_chunks == 0) continue;
            if (lane == 0) {
                if (qi > 0) mbar_wait(&bars[B_QEMPTY], (qi - 1) & 1);
                if (leader) mbar_arrive_expect_tx(&bars[B_QFULL], 2 * kQBytes);
#pragma unroll
                for (int cb = 0; cb < 2; ++cb)
                    tma_load_3d_pair_hint(sQ + cb * 128 * 128, &p.tm_q, qfull_l, cb * 64,
                                          (int)(I.it * 256 + 128 * rank), (int)I.bh, pol_stream);
            }
            ++qi;
        }
    } else if (warp == 1) {
        // ============================== MMA issuer (leader CTA, one thread)
        // Fixed order per item: S(c), S(c+1), then for each chunk j: PV(j) (after the softmax
        // of j), S(j+2).  S(j+2) reuses S_{j&1}, whose P(j) PV(j) -- issued just before, in
        // order on the tensor pipe -- has consumed.  One blocking wait at a time.
        if (leader && elect_one()) {
            int64_t c = 0;  // global chunk counter (ring stages)
            uint32_t np_[2] = {0, 0};  // P hand-offs consumed per WG (PFULL phases)
            int qi = 0, oi = 0;
            const uint32_t qa = smem_u32(sQ);
            const uint64_t qx_desc = make_sdesc(smem_u32(smem + kOffQx), 128, 256, 0);
            for (int it = 0;; ++it) {
                const int slot = it & 1;
                mbar_wait(&bars[B_IFULL + slot], (it >> 1) & 1);
                const int item = item_slot[slot];
                mbar_arrive(&bars[B_IEMPTY + slot]);
                if (item < 0) break;
                const Item I = decode(p, item);
                if (I.n_chunks == 0) continue;
                const int64_t end = c + I.n_chunks;
                mbar_wait(&bars[B_QFULL], qi & 1);
                ++qi;
                // chunk j of the item goes to WG x = j & 1 (per item, so results do not depend on
                // the dynamic schedule: every row is summed in the same order on every run)
                auto issue_s = [&](int64_t cc) {
                    const int s = (int)(cc % kStages);
                    const int x = (int)((cc - c) & 1);
                    mbar_wait(&bars[B_KFULL + s], (uint32_t)((cc / kStages) & 1));
                    tc_fence_after();
                    plan::trace(p, 2, cc);
                    const uint32_t ka = smem_u32(sK + s * kKBytes);
                    const uint32_t st = tmem_base + s_col(x);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint64_t adesc = make_sdesc(qa + (kk >> 2) * 128 * 128 + (kk & 3) * 32, 16, 1024);
                        const uint64_t bdesc = make_sdesc(ka + (kk >> 2) * kHalf * 128 + (kk & 3) * 32, 16, 1024);
                        mma2_bf16_ss(st, adesc, bdesc, kIdescS, kk > 0 ? 1u : 0u);
                    }
                    mma2_bf16_ss(st, qx_desc, make_sdesc(smem_u32(smem + kOffKx + s * kKxBytes), 128, 256, 0),
                                 kIdescS, 1u);
                    mma_commit_pair(&bars[B_SFULL + x]);
                    plan::trace(p, 12, cc);
                    mma_commit_pair(&bars[B_KEMPTY + s]);
                    if (cc == end - 1) mma_commit_pair(&bars[B_QEMPTY]);
                };
                issue_s(c);
                if (c + 1 < end) issue_s(c + 1);
                for (int64_t cc = c; cc < end; ++cc) {
                    const int s = (int)(cc % kStages);
                    const int x = (int)((cc - c) & 1);
                    mbar_wait(&bars[B_PFULL + x], np_[x] & 1u);
                    ++np_[x];
                    plan::trace(p, 5, cc);
                    if (cc == c && oi > 0) mbar_wait(&bars[B_OEMPTY], (oi - 1) & 1);  // O_0/O_1 of the last item drained
                    mbar_wait(&bars[B_VFULL + s], (uint32_t)((cc / kStages) & 1));
                    tc_fence_after();
                    const uint32_t pt = tmem_base + s_col(x);
                    const uint32_t ot = tmem_base + o_col(x);
                    const uint32_t va = smem_u32(sV + s * kVBytes);
                    const bool first = cc - c < 2;  // the item's first chunk of this WG: O_x = P V
#pragma unroll
                    for (int kk = 0; kk < kChunk / 16; ++kk) {
                        const uint64_t bdesc = make_sdesc(va + kk * 16 * 128, 128 * 128, 1024);
                        mma2_bf16_ts(ot, pt + 8u * kk, bdesc, kIdescPV, (first && kk == 0) ? 0u : 1u);
                    }
                    mma_commit_pair(&bars[B_VEMPTY + s]);
                    plan::trace(p, 4, cc);
                    if (cc + 2 < end) issue_s(cc + 2);
                }
                mma_commit_pair(&bars[B_OFIN]);
                ++oi;
                c = end;
            }
        }
        if (!leader) {
            // idle in the peer CTA: sleep on an mbarrier instead of spinning at the final cluster
            // barrier, which took issue slots from the softmax warps of the same SM sub-partitions
            mbar_wait(&bars[B_DONE], 0);
        }
        __syncwarp();
    } else {
        // ============================== loaders: kKW K warps + kVW V warps per CTA
        // Every loader warp takes part in every chunk (a few gather4s each), so a chunk's
        // gathers are issued in parallel: a warp pays a fixed ~60-110 clk per tile::gather4,
        // and one warp issuing a whole chunk (64 gather4s) made the gather latency, not the
        // ring, set the chunk period (scripts/trace_pair.py).
        //  K warp k: this CTA's K half (64 keys = 16 row groups of 4), row groups g = k (mod kKW),
        //            both column blocks, plus the groups' bias rows.
        //  V warp k: all 128 keys (32 row groups), this CTA's 64 columns, groups g = k (mod kVW).
        // Lane L handles row group g = k + kKW*L (K) / k + kVW*L (V).
        const int g = loader_index(warp);
        const bool is_k = g < kKW;
        const int k = is_k ? g : g - kKW;
        const int nw = is_k ? kKW : kVW;
        const int ngroups = is_k ? 16 : 32;
        const int grp = k + nw * (int)lane;
        const bool active = grp < ngroups;
        const int key0 = is_k ? 64 * (int)rank + 4 * grp : 4 * grp;  // first key of the row group in the chunk
        const uint32_t kfull_l0 = lbar(B_KFULL), vfull_l0 = lbar(B_VFULL);
        int64_t c = 0;
        for (int it = 0;; ++it) {
            const int slot = it & 1;
            mbar_wait_cl(&bars[B_IFULL + slot], (it >> 1) & 1);
            const int item = item_slot[slot];
            __syncwarp();
            if (lane == 0) arrive_leader(B_IEMPTY + slot);
            if (item < 0) break;
            const Item I = decode(p, item);
            if (I.n_chunks == 0) continue;
            const int64_t bq = I.bh / p.Hq, hq = I.bh % p.Hq;
            const int64_t row0 = (bq * p.Hkv + hq / (p.Hq / p.Hkv)) * p.N;
            const uint32_t* wlp = p.wl + I.base;
            auto load4 = [&](int jj, uint32_t (&e)[4]) {
                Chunk ch;
                ch.len = 0;
                ch.start = 0;
                if (jj < I.n_chunks) ch = chunk(I, jj);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int x = key0 + i;
                    e[i] = (active && x < ch.len) ? __ldcs(wlp + ch.start + x) : 0xFFFFFFFFu;  // ~0: padding
                }
            };
            uint32_t e[4];
            load4(0, e);
            for (int j = 0; j < I.n_chunks; ++j) {
                const int64_t cc = c + j;
                const int s = (int)(cc % kStages);
                const int round = (int)(cc / kStages);
                uint32_t en[4];
                load4(j + 1, en);
                int rows[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) rows[i] = (int)(row0 + (e[i] == 0xFFFFFFFFu ? 0u : (e[i] & kKeyMask)));
                if (is_k) {
                    // ---- K half: bias rows, then the gathers
                    if (round > 0) mbar_wait(&bars[B_KEMPTY + s], (round - 1) & 1);  // all lanes: no divergence
                    if (lane == 0) plan::trace(p, 0, cc);
                    __syncwarp();
                    if (active) {
                        uint8_t* kx = smem + kOffKx + s * kKxBytes;
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const uint32_t mem = e[i] == 0xFFFFFFFFu ? 0u : (e[i] >> 28);
                            const uint32_t x0 = (mem & 1u) ? 0u : 0xF180u, x1 = (mem & 2u) ? 0u : 0xF180u;
                            const uint32_t x2 = (mem & 4u) ? 0u : 0xF180u, x3 = (mem & 8u) ? 0u : 0xF180u;
                            *reinterpret_cast<uint2*>(kx + k16_offset(4 * grp + i, 0)) =
                                make_uint2(x0 | (x1 << 16), x2 | (x3 << 16));
                        }
                        fence_proxy_async();  // generic-proxy smem writes -> tcgen05.mma (async proxy)
                    }
                    __syncwarp();
                    const uint32_t kfull = kfull_l0 + 8u * (uint32_t)s;
                    if (lane == 0) {
                        if (!leader) mbar_arrive_cluster_relaxed(kfull);
                        else if (k == 0) mbar_arrive_expect_tx(&bars[B_KFULL + s], 2 * kKBytes);
                        else mbar_arrive(&bars[B_KFULL + s]);
                    }
                    if (active) {
                        uint8_t* dst = sK + s * kKBytes + 4 * grp * 128;
#pragma unroll
                        for (int cb = 0; cb < 2; ++cb)
                            tma_gather4_pair(dst + cb * kHalf * 128, &p.tm_k, kfull, cb * 64, rows[0], rows[1], rows[2],
                                             rows[3]);
                    }
                    __syncwarp();
                    if (lane == 0) plan::trace(p, 10, cc);
                } else {
                    // ---- V: this CTA's 64 columns of all 128 keys
                    if (round > 0) mbar_wait(&bars[B_VEMPTY + s], (round - 1) & 1);
                    __syncwarp();
                    const uint32_t vfull = vfull_l0 + 8u * (uint32_t)s;
                    if (lane == 0 && leader && k == 0) mbar_arrive_expect_tx(&bars[B_VFULL + s], 2 * kVBytes);
                    if (active)
                        tma_gather4_pair(sV + s * kVBytes + 4 * grp * 128, &p.tm_v, vfull, 64 * (int)rank, rows[0],
                                         rows[1], rows[2], rows[3]);
                    __syncwarp();
                    if (lane == 0 && k == 0) plan::trace(p, 11, cc);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) e[i] = en[i];
            }
            c += I.n_chunks;
        }
    }
    } else {
        setmaxnreg_inc192();
        // ============================== softmax / epilogue: WG x takes the chunks c with c & 1 == x
        const int x = ((int)warp - kSoftFirst) >> 2;
        const uint32_t quad = warp & 3u;
        const int r = (int)(quad * 32 + lane);
        const uint32_t lane_off = (quad * 32u) << 16;
        const uint32_t tS = tmem_base + lane_off + s_col(x);
        const uint32_t tO = tmem_base + lane_off + o_col(x);
        const int row_in_item = 128 * (int)rank + r;
        const float sl2 = p.scale_log2;
        const int bar_id = 1 + (int)quad;  // partner warps (same rows) of the two WGs
        const uint32_t pfull_l = lbar(B_PFULL + x);
        const uint32_t oempty_l = lbar(B_OEMPTY);
        int64_t c = 0;
        uint32_t ns = 0;  // S hand-offs consumed by this WG (SFULL_x phases)
        uint32_t fi = 0;
        for (int it = 0;; ++it) {
            const int slot = it & 1;
            mbar_wait_cl(&bars[B_IFULL + slot], (it >> 1) & 1);
            const int item = item_slot[slot];
            __syncwarp();
            if (lane == 0) arrive_leader(B_IEMPTY + slot);
            if (item < 0) break;
            const Item I = decode(p, item);
            const int64_t qrow = I.it * 256 + row_in_item;
            const bool row_ok = qrow < p.N;
            float m_ref = -INFINITY;  // log2-domain reference max (lazy rescaling)
            float2 lsum2 = make_float2(0.f, 0.f);
            int jt = 0;  // chunks of this item with this tile's keys, processed by this WG
            for (int j = 0; j < I.n_chunks; ++j) {
                const int64_t cc = c + j;
                if ((j & 1) != x) continue;
                const bool mine = (chunk(I, j).mask >> rank) & 1;
                mbar_wait(&bars[B_SFULL + x], ns & 1u);
                ++ns;
                tc_fence_after();
                if (lane == 0 && quad == 0) plan::trace(p, 6 + 2 * x, cc);
                if (!mine) {
                    tmem_st32_zero(tS);
                    tmem_st32_zero(tS + 32);
                } else {
                    // one TMEM pass: the row's 128 S columns -> registers, row max, lazy O_x
                    // rescale, P = exp2(s*scale*log2e - m) bf16-packed over S_x's first 64 columns
                    uint32_t a[128];
#pragma unroll
                    for (int qd = 0; qd < 4; ++qd) {
                        uint32_t (&aq)[32] = *reinterpret_cast<uint32_t(*)[32]>(a + 32 * qd);
                        tmem_ld32(tS + 32 * qd, aq);
                    }
                    tmem_ld_wait();
                    float mx;
                    {
                        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                        for (int t = 0; t < 128; t += 8) {
                            m4[0] = fmaxf(fmaxf(m4[0], __uint_as_float(a[t])), __uint_as_float(a[t + 1]));
                            m4[1] = fmaxf(fmaxf(m4[1], __uint_as_float(a[t + 2])), __uint_as_float(a[t + 3]));
                            m4[2] = fmaxf(fmaxf(m4[2], __uint_as_float(a[t + 4])), __uint_as_float(a[t + 5]));
                            m4[3] = fmaxf(fmaxf(m4[3], __uint_as_float(a[t + 6])), __uint_as_float(a[t + 7]));
                        }
                        mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
                    }
                    const float m_new = fmaxf(m_ref, mx * sl2);
                    const bool need = m_new > m_ref + 8.0f;
                    const float corr = need ? ex2(m_ref - m_new) : 1.0f;
                    if (need) {
                        lsum2.x *= corr;
                        lsum2.y *= corr;
                        m_ref = m_new;
                    }
                    // SFULL_x(cc): S(cc) was issued after PV(cc-2) -- this WG's previous chunk --
                    // completed, so O_x is stable here.
                    if (jt > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll
                        for (int g = 0; g < D / 8; ++g) {
                            uint32_t o[8];
                            tmem_ld8(tO + g * 8, o);
                            tmem_ld_wait();
#pragma unroll
                            for (int t = 0; t < 8; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * corr);
                            tmem_st8(tO + g * 8, o);
                        }
                    }
                    const float neg_m = (m_ref == -INFINITY) ? 0.f : -m_ref;
                    const uint64_t sl2x2 = pack_f32x2(sl2, sl2);
                    const uint64_t nmx2 = pack_f32x2(neg_m, neg_m);
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
                            // FA4-style MUFU offload: groups q % kPolyDen < kPolyNum on the FMA pipe
                            if ((t >> 2) % kPolyDen < kPolyNum) {
                                const float2 pa = ex2_poly2(xa.x, xa.y), pb = ex2_poly2(xb.x, xb.y);
                                p0 = pa.x, p1 = pa.y, p2 = pb.x, p3 = pb.y;
                            } else {
                                p0 = ex2(xa.x), p1 = ex2(xa.y), p2 = ex2(xb.x), p3 = ex2(xb.y);
                            }
                            lsum2 = fadd2(lsum2, fadd2(make_float2(p0, p1), make_float2(p2, p3)));
                            pk[t0 >> 1] = pack_bf16x2(p0, p1);
                            pk[(t0 >> 1) + 1] = pack_bf16x2(p2, p3);
                        }
                        tmem_st16(tS + 16 * qd, pk);
                    }
                    ++jt;
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0 && quad == 0) plan::trace(p, 7 + 2 * x, cc);
                if constexpr (VA_TRACE != 0) {
                    if (lane == 0 && p.trace != nullptr && blockIdx.x < 2 && cc < plan::kTraceChunks)  // debug: last warp
                        atomicMax(reinterpret_cast<unsigned long long*>(p.trace) + (15 + 16 * blockIdx.x) * plan::kTraceChunks + cc,
                                  (unsigned long long)plan::globaltimer_ns());
                }
                if (lane == 0) {
                    if (leader) mbar_arrive(&bars[B_PFULL + x]);
                    else mbar_arrive_cluster_relaxed(pfull_l);
                }
            }
            c += I.n_chunks;
            // ------------------------------------------------------------ epilogue
            // merge the two WGs' partial results of the row: side y is valid if it saw a
            // visible (member) key, i.e. m_y is not the -2^100 mask level; degenerate if none
            const bool valid = jt > 0 && m_ref >= -0x1p99f * sl2;
            const float lx = lsum2.x + lsum2.y;
            float* red = sRed;
            red[(3 * x + 0) * 128 + r] = m_ref;
            red[(3 * x + 1) * 128 + r] = lx;
            red[(3 * x + 2) * 128 + r] = valid ? 1.f : 0.f;
            named_bar_sync(bar_id, 64);
            const int y = 1 - x;
            const float m_y = red[(3 * y + 0) * 128 + r], l_y = red[(3 * y + 1) * 128 + r];
            const bool valid_y = red[(3 * y + 2) * 128 + r] != 0.f;
            named_bar_sync(bar_id, 64);  // red[] is rewritten by the next item's epilogue
            const float m_all = valid ? (valid_y ? fmaxf(m_ref, m_y) : m_ref) : (valid_y ? m_y : 0.f);
            const float w_x = valid ? ex2(m_ref - m_all) : 0.f;  // weights of O_x, O_y
            const float w_y = valid_y ? ex2(m_y - m_all) : 0.f;
            const float l = lx * w_x + l_y * w_y;
            const float inv = l > 0.f ? 1.f / l : 0.f;
            // this WG writes output columns [64x, 64x+64) from both accumulators
            __nv_bfloat16* orow = p.o + (I.bh * p.N + qrow) * D + 64 * x;
            if (I.n_chunks > 0) {
                mbar_wait(&bars[B_OFIN], fi & 1u);
                ++fi;
                tc_fence_after();
                const uint32_t tO0 = tmem_base + lane_off + o_col(x) + 64u * x;      // O_x, columns 64x..
                const uint32_t tO1 = tmem_base + lane_off + o_col(y) + 64u * x;      // O_y, columns 64x..
                const float wa = w_x * inv, wb = w_y * inv;
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    uint32_t ov[32], ow[32];
                    tmem_ld32(tO0 + 32u * g, ov);
                    tmem_ld32(tO1 + 32u * g, ow);
                    tmem_ld_wait();
                    if (row_ok && l > 0.f) {
#pragma unroll
                        for (int t = 0; t < 32; t += 8) {
                            float v8[8];
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                // a side without valid keys has weight 0; its accumulator may hold anything
                                const float fa = wa != 0.f ? __uint_as_float(ov[t + e]) * wa : 0.f;
                                const float fb = wb != 0.f ? __uint_as_float(ow[t + e]) * wb : 0.f;
                                v8[e] = fa + fb;
                            }
                            uint4 w4;
                            w4.x = pack_bf16x2(v8[0], v8[1]);
                            w4.y = pack_bf16x2(v8[2], v8[3]);
                            w4.z = pack_bf16x2(v8[4], v8[5]);
                            w4.w = pack_bf16x2(v8[6], v8[7]);
                            __stcs(reinterpret_cast<uint4*>(orow + 32 * g + t), w4);
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (leader) mbar_arrive(&bars[B_OEMPTY]);
                    else mbar_arrive_cluster_relaxed(oempty_l);
                }
            }
            if (row_ok) {
                if (l > 0.f) {
                    if (x == 0 && p.lse) p.lse[I.bh * p.N + qrow] = (m_all + __log2f(l)) * 0.69314718055994531f;
                } else {
                    // degenerate row (reading R6): O_r = V_r, LSE_r = scale*<q_r,k_r>
                    const int64_t bq = I.bh / p.Hq, hq = I.bh % p.Hq;
                    const int64_t bh_kv = bq * p.Hkv + hq / (p.Hq / p.Hkv);
                    const __nv_bfloat16* vr = p.v + (bh_kv * p.N + qrow) * D + 64 * x;
                    for (int t = 0; t < 64; ++t) orow[t] = vr[t];
                    if (x == 0) {
                        const __nv_bfloat16* kr = p.k + (bh_kv * p.N + qrow) * D;
                        const __nv_bfloat16* qr = p.q + (I.bh * p.N + qrow) * D;
                        float dot = 0.f;
                        for (int t = 0; t < D; ++t) dot = fmaf(__bfloat162float(qr[t]), __bfloat162float(kr[t]), dot);
                        if (p.lse) p.lse[I.bh * p.N + qrow] = dot * p.scale;
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_DONE]);
    }

    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair<kTmemCols>(tmem_base);
    }
}

}  // namespace pair

int grid_sms() {
    int dev = 0, sms = kNumSMsB200;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

int attn_pair_grid(int64_t items, int sms) {
    const int64_t pairs = std::min<int64_t>(items, sms / 2);
    return (int)(2 * std::max<int64_t>(1, pairs));
}

cudaError_t launch_attn_pair(const AttnParams& p, int grid, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(pair::attn_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         pair::kSmem);
    if (e != cudaSuccess) return e;
    pair::attn_pair_kernel<<<grid, pair::kThreads, pair::kSmem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace va
