// kernels.cuh — launch-side interface between the C-ABI host layer (host.cu) and
// the kernels (pool.cu, select.cu, compact.cu, attn.cu).  Internal to the library.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cuda_bf16.h>

namespace va {

constexpr int kNumSMsB200 = 148;

// ----------------------------------------------------------------------- pooling
// Eq. 2: qp[bh,i,:] = bf16_RNE( fp64 sum_{r in block i} q[bh,r,:] / h_i )
cudaError_t launch_pool(const void* q, void* qp, int64_t BH, int64_t N, int64_t D, int32_t pq,
                        cudaStream_t st);

// ----------------------------------------------------------------------- selection
enum SelectEpi : int {
    EPI_ALG1 = 0,      // Alg. 1: running max per B_K chunk, reset per group of G_K tiles
    EPI_MAX = 1,       // EXACT pass 1: row max over visible keys -> rowmax (ordered u32)
    EPI_THRESH = 2,    // EXACT pass 2: keep s >= rowmax - alpha
    EPI_TOPK_HIST = 3, // TOPK radix pass (8-bit digit `pass`)
    EPI_TOPK_EMIT = 4, // TOPK: keep key > theta, plus the first k_rem ties in index order
    EPI_SCORES = 5,    // debug: dump raw fp32 accumulators
    EPI_TK_MINMAX = 6, // TOPK window, sampled keys: row max / min -> tk_smax / tk_smin (ordered u32)
    EPI_TK_SHIST = 7,  // TOPK window, sampled keys: 256-bin histogram of round((top - s) * invw)
    EPI_TK_CAND = 8,   // TOPK window, all keys: count s > hi, collect s in [lo, hi] (whole rows)
};

struct SelectParams {
    alignas(64) CUtensorMap tm_qp;  // 3-D {D, Np, B*Hq}, box {64, 128, 1}, SW128
    alignas(64) CUtensorMap tm_k;   // 3-D {D, N, B*Hkv}, box {64, BN, 1}, SW128
    int64_t N, Np, BH, Hq, Hkv;
    int32_t pq, causal, bk, gk;
    int64_t seg_len;               // keys per CTA unit (multiple of BN and of bk*gk, or >= N)
    int64_t n_seg;                 // segments per row tile
    int64_t n_mt;                  // 128-row tiles per head
    int64_t words_per_row;         // bitmask row stride (u32 words)
    uint32_t* bitmask;             // [BH*Np, words_per_row]
    unsigned long long* counts;    // [BH*Np]
    uint32_t* rowmax;              // [BH*Np] ordered keys (EXACT)
    uint32_t* segmax;              // [BH*Np][n_seg] ordered keys: per-segment row max (split ALG1)
    int32_t split;                 // ALG1 K-split: EPI_MAX writes segmax; EPI_ALG1 starts
                                   // each segment's running max at the max of the earlier segments
    uint32_t* tk_prefix;           // [BH*Np] TOPK radix state
    uint32_t* tk_krem;             // [BH*Np]
    uint32_t* tk_hist;             // [BH*Np][256] TOPK radix histogram of the pass (summed over key segments)
    float* scores_out;             // EPI_SCORES: [BH*Np, N] fp32 (debug)
    int32_t pass;                  // TOPK pass 0..3
    int64_t topk;                  // TOPK budget
    float keep_frac;
    // TOPK window selection (select.cu "windowed TOPK"): the sampled passes run on a copy of
    // every key_stride-th K row (p.N = sampled keys, N_real = the problem's N)
    int64_t N_real;
    int32_t key_stride;            // 1, or the sampling stride of the sampled passes
    int32_t only_failed;           // EPI_TOPK_HIST / EMIT / pick: rows with tk_fail set only (fallback)
    uint32_t* tk_smax;             // [R] ordered keys of the sampled row max / min
    uint32_t* tk_smin;
    float* tk_top;                 // [R] SHIST binning: bin = round((tk_top - s) * tk_invw)
    float* tk_invw;
    float* tk_lo;                  // [R] candidate window [lo, hi]
    float* tk_hi;
    float* tk_cand;                // [R][cand_cap] window scores
    int32_t* tk_cidx;              // [R][cand_cap] their key indices (ascending within a segment slice)
    int64_t cand_cap;
    uint32_t* tk_cabove;           // [R] visible scores > hi
    uint32_t* tk_ncand;            // [R] visible scores in [lo, hi]
    uint32_t* tk_fail;             // [R] 1: the window missed the k-th largest (fallback radix)
    int* tk_nfail;                 // rows with tk_fail
    float tk_sigma;                // window half-width in binomial sigmas of the sample rank (+8 ranks)
    float tk_sigma1;               // level-1 range half-width (stride-64 sub-sample), binomial sigmas (+8)
    uint32_t* tk_sabove;           // [R] stride-8 sampled scores above the level-2 range
    float alpha_raw[1024];         // per q head: alpha / scale (raw-accumulator units)
};

cudaError_t launch_select(const SelectParams& p, int epi, int D, cudaStream_t st);
int select_bn(int epi);  // key tile (tensor-map box rows) of a selection epilogue
// TOPK: after a histogram pass, per row: the digit bin holding the k_rem-th largest remaining
// key -> tk_prefix <<= 8 | bin, tk_krem -= keys in higher bins.
cudaError_t launch_topk_pick(const SelectParams& p, cudaStream_t st);
// Windowed TOPK (few passes over sampled keys, one candidate pass, an exact select over the
// candidates; fallback to the radix passes for rows whose window missed):
// every key_stride-th row of K -> ks [B*Hkv][Ns][D]
cudaError_t launch_tk_sample_k(const void* k, void* ks, int64_t BHkv, int64_t N, int64_t Ns, int64_t D, int stride,
                               cudaStream_t st);
// stage 0: init per-row state; 1: level-1 binning from the sampled min/max; 2: level-2 binning
// inside the level-1 bin of the sampled k-th largest; 3: the candidate window [lo, hi]
cudaError_t launch_tk_rows(const SelectParams& p, int stage, int stride, cudaStream_t st);
// exact k-th largest among the window candidates -> tk_prefix / tk_krem, or tk_fail
cudaError_t launch_tk_exact(const SelectParams& p, cudaStream_t st);

// ---------------------------------------------------------------------- compaction
// offsets[r+1] = sum counts[0..r]; d_nnz = total.
cudaError_t launch_scan(const unsigned long long* counts, int64_t R, int64_t* offsets, int64_t* d_nnz,
                        cudaStream_t st);
// Emission on a side stream beside the attention kernel (one small CTA per SM).
cudaError_t launch_emit_shadow(const uint32_t* bitmask, int64_t words_per_row, const int64_t* offsets,
                               const int64_t* d_nnz, int64_t cap, int32_t* indices, int64_t BH, int64_t Np,
                               int64_t N, int32_t pq, int32_t causal, int sms, cudaStream_t st);
// Emits ascending indices of set bits of each row if *d_nnz <= cap.
cudaError_t launch_emit(const uint32_t* bitmask, int64_t words_per_row, const int64_t* offsets,
                        const int64_t* d_nnz, int64_t cap, int32_t* indices, int64_t BH, int64_t Np,
                        int64_t N, int32_t pq, int32_t causal, cudaStream_t st);

// Fused select->attend plan: the 3-segment attention worklist per 256-row item,
// straight from the selection bitmask (see compact.cu).
cudaError_t launch_plan(const uint32_t* bitmask, int64_t words_per_row, const int64_t* offsets, const int64_t* d_nnz,
                        int64_t wl_cap, uint32_t* wl, int32_t* wl_len, int64_t BH, int64_t Np, int64_t N, int32_t pq,
                        int32_t causal, cudaStream_t st);

// ------------------------------------------------------------- naive baselines (naive.cu)
// Materialise-then-filter selection (Fig. 5): row statistics, minS filter, topP
// (segmented sort + cumulative-mass cut), all on the raw fp32 score map [R, N].
cudaError_t launch_naive_row_stats(const float* scores, int64_t R, int64_t Np, int64_t N, int32_t pq, int32_t causal,
                                   float sl2, int want_z, float* rmax, double* rz, cudaStream_t st);
cudaError_t launch_naive_mins(const float* scores, int64_t R, int64_t Np, int64_t N, int32_t pq, int32_t causal,
                              const float* rmax, float alpha_raw, uint32_t* bitmask, int64_t words_per_row,
                              unsigned long long* counts, cudaStream_t st);
int64_t naive_topp_batch_rows(int64_t R, int64_t N);
size_t naive_topp_sort_temp_bytes(int64_t batch_rows, int64_t N);
cudaError_t launch_naive_topp(const float* scores, int64_t R, int64_t Np, int64_t N, int32_t pq, int32_t causal,
                              float sl2, float top_p, const float* rmax, const double* rz, float* skeys, int32_t* vals_in,
                              int32_t* vals_out, int64_t* seg_begin, int64_t* seg_end, void* temp, size_t temp_bytes,
                              uint32_t* bitmask, int64_t words_per_row, unsigned long long* counts, cudaStream_t st);

// ----------------------------------------------------------------------- attention
struct AttnParams {
    alignas(64) CUtensorMap tm_q;  // 3-D {D, N, B*Hq}, box {64, 128, 1}
    alignas(64) CUtensorMap tm_k;  // dense: 3-D {D, N, B*Hkv} box {64,128,1}; gather: 2-D {D, B*Hkv*N} box {64,1}
    alignas(64) CUtensorMap tm_v;
    const __nv_bfloat16* q;        // raw pointers for the degenerate-row fallback
    const __nv_bfloat16* k;
    const __nv_bfloat16* v;
    __nv_bfloat16* o;              // [B*Hq, N, D]
    float* lse;                    // [B*Hq, N] or null
    const uint32_t* wl;            // gather: union entries (key | membership bits << 28, bit b = block b of the item)
    const int64_t* offsets;        // gather: CSR offsets [B*Hq*Np + 1] (item base = offsets[bh*Np + (256/pq)*item])
    const int32_t* wl_len;         // gather: [B*Hq*n_mt][3] union segment lengths (both tiles | tile 0 | tile 1)
    int* work_counter;             // dynamic tile scheduler (zeroed before launch)
    const int64_t* d_nnz;          // fused path: skip all work if *d_nnz > nnz_cap (capacity protocol)
    int64_t nnz_cap;
    long long* trace;              // debug timeline [10][4096] clock64 (CTA 0) or null
    int64_t N, Np, BH, Hq, Hkv, n_mt /* 256-row items per head */, total_items;
    int32_t pq, causal;
    float scale, scale_log2;
    int32_t strict_sync;           // attn_db: wait on every ODONE phase (compute-sanitizer synccheck runs)
    const int32_t* item_order;     // gather: [total_items] item (bh*n_mt + it) for each scheduler
                                   // position (per-head longest-first; a work window's items), or
                                   // null (head-major, position order reversed within a head)
    // output replication (vecattn_forward_replicated): each O row also goes to row
    // ((b*rep_heads + rep_head0 + h)*N + r) of every rep_o[i], or once to o_mc (NVLS multicast)
    __nv_bfloat16* rep_o[8];
    __nv_bfloat16* o_mc;
    int64_t rep_head0, rep_heads;
    int32_t rep_n;
    int32_t die_mode;              // item scheduler: 0 one counter (head-major); 1/2 one counter per die
                                   // (die = smid < nsmid/2 / smid & 1), die d takes heads h = d (mod 2)
};

// Plan from a CSR; every item skips (wl_len = 0) if offsets[BH*Np] > cap (the plan buffer's capacity).
cudaError_t launch_worklist(const int64_t* offsets, const int32_t* indices, uint32_t* wl, int32_t* wl_len,
                            int64_t BH, int64_t Np, int64_t n_it, int64_t N, int32_t pq, int64_t cap,
                            cudaStream_t st);
cudaError_t launch_attn(const AttnParams& p, int D, bool gather, int grid, cudaStream_t st);
// Scheduler order of the attention items inside the work window [lo, hi) of the flattened
// items (compact.cu): head-major; within a head longest first -- by tile-chunk count
// or (by_position) by position, reversed.  order[pos] = bh*n_mt + it.  One CTA per head;
// heads with n_mt > kLptMaxItems keep position order, reversed.
constexpr int64_t kLptMaxItems = 2048;
cudaError_t launch_lpt_order(const int32_t* wl_len, int64_t BH, int64_t n_mt, int64_t lo, int64_t hi,
                             int32_t by_position, int32_t* order, cudaStream_t st);
// Non-causal sparse attention on CTA pairs (attn_pair.cu, D = 128): grid = 2 x min(items, sms/2).
int attn_pair_grid(int64_t items, int sms);
cudaError_t launch_attn_pair(const AttnParams& p, int grid, cudaStream_t st);
int grid_sms();  // SM count of the current device
// true if launch_attn runs the pair kernel for this problem (it fills its SMs: no side CTA fits)
bool attn_uses_pair(const AttnParams& p, int D, bool gather);  // false when replicas are given
// Double-buffered 64-key variant of the gather kernel (attn_db.cu), used for non-causal plans.
cudaError_t launch_attn_db(const AttnParams& p, int D, int grid, cudaStream_t st);

}  // namespace va
