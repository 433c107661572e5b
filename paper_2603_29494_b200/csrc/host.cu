// host.cu — the C ABI (include/vecattn.h): argument validation, workspace
// carving, TMA tensor-map encoding and kernel launches.  No compute happens here:
// every step of the path runs in the kernels of pool.cu / select.cu / compact.cu /
// attn.cu.
#include "../../include/vecattn.h"
#include "kernels.cuh"

#include <cudaTypedefs.h>
#include <math.h>
#include <mutex>
#include <vector>
#include <limits>
#include <cmath>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

namespace {

using va::AttnParams;
using va::SelectParams;

constexpr size_t kAlign = 256;
constexpr int64_t kMaxSplit = 8;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    std::call_once(g_encode_once, [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    return g_encode;
}

// bf16 tensor [d2][d1][d0] (d0 innermost), box {64, box1, 1}, 128B swizzle, OOB -> 0.
bool tmap_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t box1) {
    auto enc = encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {d0 * 2, d0 * d1 * 2};
    cuuint32_t box[3] = {64, box1, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// bf16 rows [rows][d0], box {64, 1} for tile::gather4 (4 rows per instruction).
bool tmap_gather(CUtensorMap* m, const void* base, uint64_t d0, uint64_t rows) {
    auto enc = encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {d0, rows};
    cuuint64_t strides[1] = {d0 * 2};
    cuuint32_t box[2] = {64, 1};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool aligned16(const void* ptr) { return ((uintptr_t)ptr & 15u) == 0; }

vecattn_status_t check_problem(const vecattn_problem_t* p) {
    if (!p) return VECATTN_ERR_INVALID_ARGUMENT;
    if (p->B < 1 || p->Hq < 1 || p->Hkv < 1 || p->N < 1) return VECATTN_ERR_SHAPE;
    if (p->D != 64 && p->D != 128) return VECATTN_ERR_SHAPE;
    if (p->N >= (int64_t(1) << 28) || p->Hq > 1024) return VECATTN_ERR_SHAPE;
    if (p->B * p->Hkv * p->N >= (int64_t(1) << 31) || p->B * p->Hq * p->N >= (int64_t(1) << 31))
        return VECATTN_ERR_SHAPE;
    if (p->Hq % p->Hkv != 0) return VECATTN_ERR_INVALID_ARGUMENT;
    if (!(p->scale >= 0.f) || isinf(p->scale)) return VECATTN_ERR_INVALID_ARGUMENT;
    return VECATTN_OK;
}

float eff_scale(const vecattn_problem_t* p) { return p->scale > 0.f ? p->scale : 1.0f / sqrtf((float)p->D); }

int64_t n_pooled(const vecattn_problem_t* p, int32_t pq) { return (p->N + pq - 1) / pq; }

int64_t words_per_row(const vecattn_problem_t* p) { return (p->N + 255) / 256 * 8; }

vecattn_status_t check_select(const vecattn_problem_t* p, const vecattn_select_params_t* s) {
    vecattn_status_t st = check_problem(p);
    if (st != VECATTN_OK) return st;
    if (!s) return VECATTN_ERR_INVALID_ARGUMENT;
    if (s->pq != 64 && s->pq != 128) return VECATTN_ERR_INVALID_ARGUMENT;
    if (s->mode < 0 || s->mode > 2) return VECATTN_ERR_INVALID_ARGUMENT;
    if (s->mode == VECATTN_SEL_MINS_ALG1 && s->bk != 8 && s->bk != 16 && s->bk != 32 &&
        s->bk != 64 && s->bk != 128 && s->bk != 256)
        return VECATTN_ERR_INVALID_ARGUMENT;
    if (s->mode == VECATTN_SEL_MINS_ALG1 && s->gk < 1) return VECATTN_ERR_INVALID_ARGUMENT;
    if (s->mode != VECATTN_SEL_TOPK) {
        if (!(s->alpha >= 0.f) || isinf(s->alpha)) return VECATTN_ERR_INVALID_ARGUMENT;
        if (s->alpha_per_head)
            for (int64_t h = 0; h < p->Hq; ++h)
                if (!(s->alpha_per_head[h] >= 0.f) || isinf(s->alpha_per_head[h])) return VECATTN_ERR_INVALID_ARGUMENT;
    } else {
        if (s->topk <= 0 && !(s->keep_frac > 0.f && s->keep_frac <= 1.f)) return VECATTN_ERR_INVALID_ARGUMENT;
    }
    return VECATTN_OK;
}

struct SelectWs {
    void* qp;
    uint32_t* bitmask;
    unsigned long long* counts;
    uint32_t* rowmax;
    uint32_t* segmax;
    uint32_t* tk_prefix;
    uint32_t* tk_krem;
    uint32_t* tk_hist;
    // windowed TOPK (mode TOPK only)
    void* ks;            // sampled K rows [B*Hkv][Ns][D]
    void* ks1;           // level-1 sub-sample [B*Hkv][Ns1][D] (1 in kTkStride * kTkSub)
    uint32_t *tk_smax, *tk_smin, *tk_cabove, *tk_ncand, *tk_fail, *tk_sabove;
    float *tk_top, *tk_invw, *tk_lo, *tk_hi, *tk_cand;
    int32_t* tk_cidx;
    int* tk_nfail;
    int64_t cand_cap;
    size_t total;
};

constexpr int kTkStride = 8;         // windowed TOPK: 1 of every 8 keys in the sampled passes
constexpr int kTkSub = 8;            // level 1 (min/max, coarse histogram): every 8th sampled key
constexpr int64_t kTkCandSeg = 16384;  // candidate pass key segment
// a multiple of 128: the per-(segment, warp set) slices start 16-B aligned (vector candidate stores)
int64_t tk_cand_cap(const vecattn_problem_t* p) { return (std::min<int64_t>(p->N, 16384) + 127) / 128 * 128; }

SelectWs carve_select(const vecattn_problem_t* p, int32_t pq, void* base, bool topk = false) {
    const int64_t BH = p->B * p->Hq, Np = n_pooled(p, pq), R = BH * Np;
    uint8_t* b = static_cast<uint8_t*>(base);
    size_t off = 0;
    SelectWs w;
    w.qp = b + off;
    off += align_up((size_t)R * p->D * 2);
    w.bitmask = reinterpret_cast<uint32_t*>(b + off);
    off += align_up((size_t)R * words_per_row(p) * 4);
    w.counts = reinterpret_cast<unsigned long long*>(b + off);
    off += align_up((size_t)R * 8);
    w.rowmax = reinterpret_cast<uint32_t*>(b + off);
    off += align_up((size_t)R * 4);
    w.segmax = reinterpret_cast<uint32_t*>(b + off);
    off += align_up((size_t)R * kMaxSplit * 4);
    w.tk_prefix = reinterpret_cast<uint32_t*>(b + off);
    off += align_up((size_t)R * 4);
    w.tk_krem = reinterpret_cast<uint32_t*>(b + off);
    off += align_up((size_t)R * 4);
    w.tk_hist = reinterpret_cast<uint32_t*>(b + off);
    off += align_up((size_t)R * 256 * 4 * (topk ? 2 : 1));  // windowed TOPK: two histogram levels
    w.ks = w.ks1 = nullptr;
    w.tk_smax = w.tk_smin = w.tk_cabove = w.tk_ncand = w.tk_fail = w.tk_sabove = nullptr;
    w.tk_top = w.tk_invw = w.tk_lo = w.tk_hi = w.tk_cand = nullptr;
    w.tk_cidx = nullptr;
    w.tk_nfail = nullptr;
    w.cand_cap = 0;
    if (topk) {
        const int64_t Ns = (p->N + kTkStride - 1) / kTkStride;
        w.ks = b + off;
        off += align_up((size_t)(p->B * p->Hkv * Ns * p->D * 2));
        const int64_t Ns1 = (p->N + kTkStride * kTkSub - 1) / (kTkStride * kTkSub);
        w.ks1 = b + off;
        off += align_up((size_t)(p->B * p->Hkv * Ns1 * p->D * 2));
        uint32_t** u32s[] = {&w.tk_smax, &w.tk_smin, &w.tk_cabove, &w.tk_fail, &w.tk_sabove};
        for (uint32_t** x : u32s) {
            *x = reinterpret_cast<uint32_t*>(b + off);
            off += align_up((size_t)R * 4);
        }
        w.tk_ncand = reinterpret_cast<uint32_t*>(b + off);  // [R][candidate-pass segments]
        off += align_up((size_t)R * 4 * 2 * (size_t)((p->N + kTkCandSeg - 1) / kTkCandSeg));  // x 2 warp sets
        float** f32s[] = {&w.tk_top, &w.tk_invw, &w.tk_lo, &w.tk_hi};
        for (float** x : f32s) {
            *x = reinterpret_cast<float*>(b + off);
            off += align_up((size_t)R * 4);
        }
        w.tk_nfail = reinterpret_cast<int*>(b + off);
        off += align_up(16);
        w.cand_cap = tk_cand_cap(p);
        w.tk_cand = reinterpret_cast<float*>(b + off);
        off += align_up((size_t)R * (size_t)w.cand_cap * 4);
        w.tk_cidx = reinterpret_cast<int32_t*>(b + off);
        off += align_up((size_t)R * (size_t)w.cand_cap * 4);
    }
    w.total = off;
    return w;
}

int64_t gcd64(int64_t a, int64_t b) { return b == 0 ? a : gcd64(b, a % b); }

// ALG1 K-split.  With G_K * B_K >= N (DiT: one Alg. 1 group per row) a row is
// one sequential unit, so few heads per GPU leave SMs idle (3 heads at 8 GPUs = 48 row tiles
// for 148 SMs).  Then split rows into up to kMaxSplit key segments: a max pass writes each
// segment's row max, and the ALG1 pass starts segment s at the max of segments < s, which is
// exactly the running max Alg. 1 carries into the segment.  Returns the segment count (1 = no
// split).  VECATTN_SELECT_SPLIT=<n> forces n (tests).
int select_split(const vecattn_problem_t* p, const vecattn_select_params_t* s, int64_t units) {
    const int64_t G = (int64_t)s->bk * (int64_t)s->gk;
    if (s->mode != VECATTN_SEL_MINS_ALG1 || p->causal || G < p->N) return 1;
    int n = 1;
    if (const char* env = getenv("VECATTN_SELECT_SPLIT")) n = atoi(env);
    else {
        int dev = 0, sms = va::kNumSMsB200;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (units < sms) n = (int)((sms + units - 1) / units);  // fill one wave
    }
    n = std::max(1, std::min(n, (int)kMaxSplit));
    const int64_t nblk = (p->N + 255) / 256;  // segments are multiples of the 256-key tile
    return (int)std::min<int64_t>(n, nblk);
}

// Keys per CTA unit.  Units never split a G_K group (Alg. 1 running max scope), so a
// segment is a multiple of lcm(B_K*G_K, 256); TOPK needs whole rows.
void plan_segments(const vecattn_problem_t* p, const vecattn_select_params_t* s, int epi, SelectParams& sp) {
    const int64_t Nr = (p->N + 255) / 256 * 256;
    int64_t seg = Nr;
    if (epi == va::EPI_ALG1) {
        const int64_t G = (int64_t)s->bk * (int64_t)s->gk;
        if (G < p->N) {
            const int64_t L = G / gcd64(G, 256) * 256;
            if (L < p->N) seg = L * std::max<int64_t>(1, 16384 / L);
        }
    } else if (epi == va::EPI_MAX || epi == va::EPI_THRESH || epi == va::EPI_SCORES || epi == va::EPI_TOPK_HIST) {
        seg = 16384;  // TOPK histogram passes: per-segment histograms are summed in tk_hist
    }
    if (epi == va::EPI_TK_CAND) seg = std::min<int64_t>(Nr, kTkCandSeg);  // per-(row, segment) candidate slices
    if (seg > Nr) seg = Nr;
    // few rows (e.g. one GPU's share of the heads): shorter segments until the units fill
    // two waves, keeping segments a multiple of the unit granule and >= 2048 keys
    const int64_t granule = (epi == va::EPI_ALG1 && (int64_t)s->bk * s->gk < p->N)
                                ? (int64_t)s->bk * s->gk / gcd64((int64_t)s->bk * s->gk, 256) * 256
                                : 256;
    const int64_t row_units = sp.BH * sp.n_mt;
    if (epi == va::EPI_ALG1 || epi == va::EPI_MAX || epi == va::EPI_THRESH) {
        while (row_units * ((p->N + seg - 1) / seg) < 2 * va::kNumSMsB200 && seg / 2 >= 2048 &&
               (seg / 2) % granule == 0 && (epi != va::EPI_ALG1 || (int64_t)s->bk * s->gk < p->N))
            seg /= 2;
    }
    sp.seg_len = seg;
    sp.n_seg = (p->N + seg - 1) / seg;
}

vecattn_status_t fill_select_params(const vecattn_problem_t* p, const vecattn_select_params_t* s, int32_t pq,
                                    const void* k, const SelectWs& w, SelectParams& sp) {
    memset(&sp, 0, sizeof(sp));
    const int64_t BH = p->B * p->Hq, Np = n_pooled(p, pq);
    sp.N = p->N;
    sp.Np = Np;
    sp.BH = BH;
    sp.Hq = p->Hq;
    sp.Hkv = p->Hkv;
    sp.pq = pq;
    sp.causal = p->causal ? 1 : 0;
    sp.bk = s ? s->bk : 16;
    sp.gk = s ? s->gk : 1;
    sp.n_mt = (Np + 127) / 128;
    sp.words_per_row = words_per_row(p);
    sp.bitmask = w.bitmask;
    sp.counts = w.counts;
    sp.rowmax = w.rowmax;
    sp.segmax = w.segmax;
    sp.tk_prefix = w.tk_prefix;
    sp.tk_krem = w.tk_krem;
    sp.tk_hist = w.tk_hist;
    sp.N_real = p->N;
    sp.key_stride = 1;
    sp.only_failed = 0;
    sp.tk_smax = w.tk_smax;
    sp.tk_smin = w.tk_smin;
    sp.tk_top = w.tk_top;
    sp.tk_invw = w.tk_invw;
    sp.tk_lo = w.tk_lo;
    sp.tk_hi = w.tk_hi;
    sp.tk_cand = w.tk_cand;
    sp.tk_cidx = w.tk_cidx;
    sp.cand_cap = w.cand_cap;
    sp.tk_cabove = w.tk_cabove;
    sp.tk_ncand = w.tk_ncand;
    sp.tk_fail = w.tk_fail;
    sp.tk_nfail = w.tk_nfail;
    sp.tk_sigma = 4.5f;
    sp.tk_sigma1 = 8.0f;
    sp.tk_sabove = w.tk_sabove;
    if (const char* ev = getenv("VECATTN_TOPK_SIGMA")) sp.tk_sigma = (float)atof(ev);  // experiments (scripts)
    sp.topk = s ? s->topk : 0;
    sp.keep_frac = s ? s->keep_frac : 0.f;
    const float scale = eff_scale(p);
    for (int64_t h = 0; h < p->Hq; ++h) {
        const float a = s ? (s->alpha_per_head ? s->alpha_per_head[h] : s->alpha) : 0.f;
        sp.alpha_raw[h] = a / scale;
    }
    if (!tmap_3d(&sp.tm_qp, w.qp, (uint64_t)p->D, (uint64_t)Np, (uint64_t)BH, 128)) return VECATTN_ERR_UNSUPPORTED;
    return VECATTN_OK;
}

vecattn_status_t set_k_map(const vecattn_problem_t* p, const void* k, int bn, SelectParams& sp) {
    if (!tmap_3d(&sp.tm_k, k, (uint64_t)p->D, (uint64_t)p->N, (uint64_t)(p->B * p->Hkv), (uint32_t)bn))
        return VECATTN_ERR_UNSUPPORTED;
    return VECATTN_OK;
}

thread_local cudaError_t g_last_cuda_error = cudaSuccess;

vecattn_status_t cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return VECATTN_OK;
    g_last_cuda_error = e;
    return VECATTN_ERR_CUDA;
}


// Pooling + the selection GEMM passes of the configured mode + scan (counts -> offsets).
cudaError_t run_select(const vecattn_problem_t* p, const vecattn_select_params_t* s, const void* q, const void* k,
                       int64_t* offsets, int64_t* d_nnz, const SelectWs& w, SelectParams& sp, cudaStream_t cs) {
    const int64_t R = sp.BH * sp.Np;
    const int nsplit = select_split(p, s, sp.BH * sp.n_mt);
    auto run = [&](int epi, int pass) -> cudaError_t {
        plan_segments(p, s, epi, sp);
        sp.split = 0;
        if (nsplit > 1 && (epi == va::EPI_ALG1 || epi == va::EPI_MAX)) {
            const int64_t nblk = (p->N + 255) / 256;
            sp.seg_len = (nblk + nsplit - 1) / nsplit * 256;
            sp.n_seg = (p->N + sp.seg_len - 1) / sp.seg_len;
            sp.split = 1;
        }
        sp.pass = pass;
        if (set_k_map(p, k, va::select_bn(epi), sp) != VECATTN_OK) return cudaErrorInvalidValue;
        return va::launch_select(sp, epi, (int)p->D, cs);
    };
    cudaError_t e = va::launch_pool(q, w.qp, sp.BH, p->N, p->D, s->pq, cs);
    if (e == cudaSuccess) e = cudaMemsetAsync(w.counts, 0, (size_t)R * 8, cs);
    if (e == cudaSuccess) {
        if (s->mode == VECATTN_SEL_MINS_ALG1) {
            if (nsplit > 1) e = run(va::EPI_MAX, 0);  // per-segment row maxima (split)
            if (e == cudaSuccess) e = run(va::EPI_ALG1, 0);
        } else if (s->mode == VECATTN_SEL_MINS_EXACT) {
            e = cudaMemsetAsync(w.rowmax, 0, (size_t)R * 4, cs);
            if (e == cudaSuccess) e = run(va::EPI_MAX, 0);
            if (e == cudaSuccess) e = run(va::EPI_THRESH, 0);
        } else {
            // windowed TOPK (select.cu): sampled passes -> window -> one candidate pass -> exact
            // select; the radix passes below then run only for rows whose window missed
            // (VECATTN_TOPK_RADIX=1: radix passes for every row, the previous method)
            const bool windowed = w.tk_cand != nullptr && !getenv("VECATTN_TOPK_RADIX");
            if (windowed) {
                const int64_t Ns = (p->N + kTkStride - 1) / kTkStride;
                // level 1 gets its own hashed-offset sample (every 8th row of the 1-in-8 sample
                // would sit at a fixed phase of period-64 structure, e.g. 64-wide video frames)
                const int64_t Ns1 = (p->N + kTkStride * kTkSub - 1) / (kTkStride * kTkSub);
                e = va::launch_tk_sample_k(k, w.ks, p->B * p->Hkv, p->N, Ns, p->D, kTkStride, cs);
                if (e == cudaSuccess)
                    e = va::launch_tk_sample_k(k, w.ks1, p->B * p->Hkv, p->N, Ns1, p->D, kTkStride * kTkSub, cs);
                if (e == cudaSuccess) e = va::launch_tk_rows(sp, 0, kTkStride, cs);
                if (e == cudaSuccess) e = cudaMemsetAsync(w.tk_nfail, 0, sizeof(int), cs);
                // sampled passes: K = one row per kTkStride (hashed offsets); level 1 (min/max and
                // the coarse histogram that places level 2): one per kTkStride * kTkSub
                SelectParams* ss = new SelectParams(sp);
                auto run_sampled = [&](int epi, int pass, bool level1) -> cudaError_t {
                    const int64_t n = level1 ? Ns1 : Ns;
                    ss->N = n;
                    ss->key_stride = level1 ? kTkStride * kTkSub : kTkStride;
                    plan_segments(p, s, epi, *ss);
                    // min/max: 4096-key units (atomics merge them); histograms: whole sampled rows
                    ss->seg_len = epi == va::EPI_TK_SHIST ? (n + 255) / 256 * 256
                                                          : std::min<int64_t>(4096, (n + 255) / 256 * 256);
                    ss->n_seg = (n + ss->seg_len - 1) / ss->seg_len;
                    ss->split = 0;
                    ss->pass = pass;
                    if (!tmap_3d(&ss->tm_k, level1 ? w.ks1 : w.ks, (uint64_t)p->D, (uint64_t)n, (uint64_t)(p->B * p->Hkv),
                                 (uint32_t)va::select_bn(epi)))
                        return cudaErrorInvalidValue;
                    return va::launch_select(*ss, epi, (int)p->D, cs);
                };
                if (e == cudaSuccess) e = run_sampled(va::EPI_TK_MINMAX, 0, true);
                if (e == cudaSuccess) e = va::launch_tk_rows(sp, 1, kTkStride * kTkSub, cs);
                if (e == cudaSuccess) e = cudaMemsetAsync(w.tk_hist, 0, (size_t)R * 256 * 4 * 2, cs);
                if (e == cudaSuccess) e = run_sampled(va::EPI_TK_SHIST, 0, true);
                if (e == cudaSuccess) e = va::launch_tk_rows(sp, 2, kTkStride * kTkSub, cs);
                if (e == cudaSuccess) e = run_sampled(va::EPI_TK_SHIST, 1, false);
                if (e == cudaSuccess) e = va::launch_tk_rows(sp, 3, kTkStride, cs);
                delete ss;
                // VECATTN_TOPK_FORCE_FALLBACK=1 (tests): no candidate room -> every row takes the
                // radix fallback, which must give the same selection
                // candidate counts of every (row, segment, warp set) slice: causal units above
                // the diagonal never run, so their slices must read as empty
#ifndef VA_TEST_NO_NCAND_CLEAR  // (build knob used once to check that tests/test_gpu_stale_ws.py catches the stale read)
                if (e == cudaSuccess)
                    e = cudaMemsetAsync(w.tk_ncand, 0, (size_t)R * 4 * 2 * (size_t)((p->N + kTkCandSeg - 1) / kTkCandSeg), cs);
#endif
                const int64_t cap_keep = sp.cand_cap;
                if (getenv("VECATTN_TOPK_FORCE_FALLBACK")) sp.cand_cap = 0;
                if (e == cudaSuccess) e = run(va::EPI_TK_CAND, 0);
                if (e == cudaSuccess) e = va::launch_tk_exact(sp, cs);
                sp.cand_cap = cap_keep;
                if (e == cudaSuccess && getenv("VECATTN_TOPK_DEBUG")) {  // diagnostics (scripts only)
                    cudaStreamSynchronize(cs);
                    const int64_t nsg = 2 * ((p->N + kTkCandSeg - 1) / kTkCandSeg);
                    std::vector<uint32_t> ab(R), nc(R), fl(R), ncs(R * nsg);
                    std::vector<float> lo(R), hi(R);
                    int nf = 0;
                    cudaMemcpy(ab.data(), w.tk_cabove, R * 4, cudaMemcpyDeviceToHost);
                    cudaMemcpy(ncs.data(), w.tk_ncand, R * nsg * 4, cudaMemcpyDeviceToHost);
                    for (int64_t r = 0; r < R; ++r) {
                        nc[r] = 0;
                        for (int64_t g = 0; g < nsg; ++g) nc[r] += ncs[r * nsg + g];
                    }
                    cudaMemcpy(fl.data(), w.tk_fail, R * 4, cudaMemcpyDeviceToHost);
                    cudaMemcpy(lo.data(), w.tk_lo, R * 4, cudaMemcpyDeviceToHost);
                    cudaMemcpy(hi.data(), w.tk_hi, R * 4, cudaMemcpyDeviceToHost);
                    cudaMemcpy(&nf, w.tk_nfail, 4, cudaMemcpyDeviceToHost);
                    double sn = 0;
                    uint32_t mx = 0, over = 0;
                    for (int64_t r = 0; r < R; ++r) {
                        sn += nc[r];
                        mx = std::max(mx, nc[r]);
                        over += nc[r] > (uint32_t)w.cand_cap;
                    }
                    uint64_t hsh = 1469598103934665603ull;  // FNV-1a of the window bounds' bits
                    for (int64_t r = 0; r < R; ++r) {
                        uint32_t b2[2];
                        memcpy(&b2[0], &lo[r], 4);
                        memcpy(&b2[1], &hi[r], 4);
                        hsh = (hsh ^ b2[0]) * 1099511628211ull;
                        hsh = (hsh ^ b2[1]) * 1099511628211ull;
                    }
                    fprintf(stderr, "[topk window] rows %lld failed %d overflow %u mean cand %.0f max %u window hash %016llx\n",
                            (long long)R, nf, over, sn / R, mx, (unsigned long long)hsh);
                    std::vector<uint32_t> smx(4), smn(4), h(512);
                    std::vector<float> tp(4), iw(4);
                    cudaMemcpy(smx.data(), w.tk_smax, 16, cudaMemcpyDeviceToHost);
                    cudaMemcpy(smn.data(), w.tk_smin, 16, cudaMemcpyDeviceToHost);
                    cudaMemcpy(tp.data(), w.tk_top, 16, cudaMemcpyDeviceToHost);
                    cudaMemcpy(iw.data(), w.tk_invw, 16, cudaMemcpyDeviceToHost);
                    cudaMemcpy(h.data(), w.tk_hist, 256 * 4, cudaMemcpyDeviceToHost);
                    cudaMemcpy(h.data() + 256, w.tk_hist + (size_t)R * 256, 256 * 4, cudaMemcpyDeviceToHost);
                    uint64_t s1 = 0, s2 = 0;
                    for (int x = 0; x < 256; ++x) { s1 += h[x]; s2 += h[256 + x]; }
                    fprintf(stderr, "  row0 smax %08x smin %08x top2 %g invw2 %g hist1 sum %llu hist2 sum %llu\n", smx[0], smn[0],
                            tp[0], iw[0], (unsigned long long)s1, (unsigned long long)s2);
                    for (int64_t r = 0; r < R; ++r)
                        if (fl[r]) {  // dump the first failed row's sample histograms (scripts/topk_window_dbg.py)
                            std::vector<uint32_t> hh(512), mm(2);
                            std::vector<float> tt(2);
                            cudaMemcpy(hh.data(), w.tk_hist + r * 256, 1024, cudaMemcpyDeviceToHost);
                            cudaMemcpy(hh.data() + 256, w.tk_hist + (R + r) * 256, 1024, cudaMemcpyDeviceToHost);
                            cudaMemcpy(&mm[0], w.tk_smax + r, 4, cudaMemcpyDeviceToHost);
                            cudaMemcpy(&mm[1], w.tk_smin + r, 4, cudaMemcpyDeviceToHost);
                            cudaMemcpy(&tt[0], w.tk_top + r, 4, cudaMemcpyDeviceToHost);
                            cudaMemcpy(&tt[1], w.tk_invw + r, 4, cudaMemcpyDeviceToHost);
                            if (FILE* fo = fopen("gpurun_out/topk_fail_row.bin", "wb")) {
                                fwrite(hh.data(), 4, 512, fo);
                                fwrite(mm.data(), 4, 2, fo);
                                fwrite(tt.data(), 4, 2, fo);
                                fwrite(&lo[r], 4, 1, fo);
                                fwrite(&hi[r], 4, 1, fo);
                                fwrite(&ab[r], 4, 1, fo);
                                fwrite(&nc[r], 4, 1, fo);
                                fclose(fo);
                            }
                            break;
                        }
                    int shown = 0;
                    for (int64_t r = 0; r < R && shown < 8; ++r)
                        if (fl[r]) {
                            ++shown;
                            fprintf(stderr, "  FAILED row %lld (i %lld) above %u ncand %u lo %g hi %g\n", (long long)r,
                                    (long long)(r % sp.Np), ab[r], nc[r], lo[r], hi[r]);
                        }
                }
                sp.only_failed = 1;  // fallback: radix passes for the rows the window missed
            }
            for (int pass = 0; pass < 4 && e == cudaSuccess; ++pass) {
                e = cudaMemsetAsync(w.tk_hist, 0, (size_t)R * 256 * 4, cs);
                if (e == cudaSuccess) e = run(va::EPI_TOPK_HIST, pass);
                if (e == cudaSuccess) e = va::launch_topk_pick(sp, cs);
            }
            // windowed rows already have their bits (the candidate pass wrote the keys above the
            // window, the exact select the kept candidates) and counts = k; the emit pass runs
            // for the fallback rows only
            if (e == cudaSuccess) e = run(va::EPI_TOPK_EMIT, 0);
            sp.only_failed = 0;
        }
    }
    if (e == cudaSuccess) e = va::launch_scan(w.counts, R, offsets, d_nnz, cs);
    return e;
}

#define VA_CU(x)                                            \
    do {                                                    \
        cudaError_t e_ = (x);                               \
        if (e_ != cudaSuccess) return cuda_status(e_);      \
    } while (0)

__global__ void validate_kernel(const int64_t* __restrict__ offsets, const int32_t* __restrict__ indices,
                                int64_t R, int64_t Np, int64_t N, int32_t pq, int32_t causal, int32_t* d_bad) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const int64_t i = r % Np;
    const int64_t lim = causal ? std::min<int64_t>(N, (i + 1) * (int64_t)pq) : N;  // exclusive
    const int64_t a = offsets[r], b = offsets[r + 1];
    bool bad = b < a;
    int64_t prev = -1;
    for (int64_t t = a; t < b && !bad; ++t) {
        const int64_t j = indices[t];
        if (j <= prev || j < 0 || j >= lim) bad = true;
        prev = j;
    }
    if (bad) atomicAdd(d_bad, 1);
}

}  // namespace

namespace {
// Library-owned side stream per device for the emission that runs beside the attention
// kernel, with its fork/join events.  Created once; the mutex serialises the
// record -> wait -> launch -> record -> wait sequence of concurrent host callers.
struct SideStream {
    std::mutex mu;
    cudaStream_t s = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int sms = va::kNumSMsB200;
};
SideStream g_side[64];
std::mutex g_side_init;
SideStream* side_stream() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> g(g_side_init);
    SideStream& x = g_side[dev];
    if (!x.s) {
        if (cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        cudaEventCreateWithFlags(&x.ev_fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&x.ev_join, cudaEventDisableTiming);
        cudaDeviceGetAttribute(&x.sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return &x;
}
}  // namespace

extern "C" {

int32_t vecattn_abi_version(void) { return 1; }

// ------------------------------------------------------------------ measurement hook
namespace {
struct Timing {
    bool enabled = false;
    bool created = false;
    bool has_sel = false, has_plan = false, has_attn = false;
    cudaEvent_t ev[4];  // select start, select end / plan start, plan end / attn start, attn end
};
Timing g_timing;
void tmark(int i, cudaStream_t st) {
    if (g_timing.enabled) cudaEventRecord(g_timing.ev[i], st);
}
void tbegin(bool sel, bool plan) {
    g_timing.has_sel = sel;
    g_timing.has_plan = plan;
    g_timing.has_attn = true;
}
}  // namespace

vecattn_status_t vecattn_kernel_timing(int32_t enable) {
    if (enable && !g_timing.created) {
        for (auto& e : g_timing.ev)
            if (cudaEventCreate(&e) != cudaSuccess) return cuda_status(cudaGetLastError());
        g_timing.created = true;
    }
    g_timing.enabled = enable != 0;
    return VECATTN_OK;
}

vecattn_status_t vecattn_kernel_timing_last(float* select_ms, float* plan_ms, float* attn_ms) {
    if (!select_ms || !plan_ms || !attn_ms) return VECATTN_ERR_INVALID_ARGUMENT;
    *select_ms = *plan_ms = *attn_ms = -1.f;
    if (!g_timing.created) return VECATTN_OK;
    if (cudaEventSynchronize(g_timing.ev[3]) != cudaSuccess) return cuda_status(cudaGetLastError());
    if (g_timing.has_sel) cudaEventElapsedTime(select_ms, g_timing.ev[0], g_timing.ev[1]);
    if (g_timing.has_plan) cudaEventElapsedTime(plan_ms, g_timing.ev[1], g_timing.ev[2]);
    if (g_timing.has_attn) cudaEventElapsedTime(attn_ms, g_timing.ev[2], g_timing.ev[3]);
    return VECATTN_OK;
}

// ------------------------------------------------------------ per-head filter ratios (Eq. 4)
// Eq. 4 run backwards over heads on the quantised sparsity sum s (capped at the
// target, since any sum >= target is equivalent): F[h][s] = best performance of heads
// h..H-1 given the sum s of heads 0..h-1; F[H][s] = 0 if s >= need else -inf.  The forward
// reconstruction takes the smallest candidate attaining F at every head.
vecattn_status_t vecattn_alpha_dp(int32_t H, int32_t n_cand, const float* sp, const float* perf, float rho_target,
                                  int32_t grid, int32_t* choice, double* best) {
    if (!sp || !perf || !choice || !best || H < 1 || n_cand < 1 || grid < 1 || !(rho_target >= 0.f) ||
        !(rho_target <= 1.f))
        return VECATTN_ERR_INVALID_ARGUMENT;
    const int64_t C = n_cand;
    std::vector<int64_t> q((size_t)H * C);
    for (int64_t x = 0; x < (int64_t)H * C; ++x) {
        if (!std::isfinite(sp[x]) || !std::isfinite(perf[x]) || sp[x] < 0.f || sp[x] > 1.f)
            return VECATTN_ERR_INVALID_ARGUMENT;
        q[x] = (int64_t)std::floor((double)sp[x] * grid + 0.5);
    }
    const int64_t need = (int64_t)std::floor((double)rho_target * grid * H + 0.5);
    const double NEG = -std::numeric_limits<double>::infinity();
    std::vector<double> F((size_t)(H + 1) * (need + 1), NEG);
    auto at = [&](int64_t h, int64_t s) -> double& { return F[(size_t)h * (need + 1) + s]; };
    at(H, need) = 0.0;
    for (int64_t h = H - 1; h >= 0; --h)
        for (int64_t s = 0; s <= need; ++s) {
            double bestv = NEG;
            for (int64_t c = 0; c < C; ++c) {
                const double nxt = at(h + 1, std::min(need, s + q[h * C + c]));
                if (nxt == NEG) continue;
                bestv = std::max(bestv, (double)perf[h * C + c] + nxt);
            }
            at(h, s) = bestv;
        }
    *best = at(0, 0);
    if (*best == NEG) return VECATTN_ERR_INVALID_ARGUMENT;
    int64_t s = 0;
    for (int64_t h = 0; h < H; ++h)
        for (int64_t c = 0; c < C; ++c) {
            const int64_t s2 = std::min(need, s + q[h * C + c]);
            const double nxt = at(h + 1, s2);
            if (nxt != NEG && (double)perf[h * C + c] + nxt == at(h, s)) {
                choice[h] = (int32_t)c;
                s = s2;
                break;
            }
        }
    return VECATTN_OK;
}

// ------------------------------------------------------------ naive selection baselines
namespace {
struct NaiveWs {
    float* scores;
    float* rmax;
    double* rz;
    float* skeys;
    int32_t* vals_in;
    int32_t* vals_out;
    int64_t* seg_begin;
    int64_t* seg_end;
    void* temp;
    size_t temp_bytes;
    size_t total;
};
NaiveWs carve_naive(const vecattn_problem_t* p, int32_t pq, int32_t mode, void* base) {
    const int64_t R = p->B * p->Hq * n_pooled(p, pq), N = p->N;
    uint8_t* b = static_cast<uint8_t*>(base);
    NaiveWs w;
    memset(&w, 0, sizeof(w));
    size_t off = 0;
    auto take = [&](size_t bytes) {
        uint8_t* x = b ? b + off : nullptr;
        off += align_up(bytes);
        return x;
    };
    w.scores = reinterpret_cast<float*>(take((size_t)R * N * 4));
    w.rmax = reinterpret_cast<float*>(take((size_t)R * 4));
    w.rz = reinterpret_cast<double*>(take((size_t)R * 8));
    if (mode == VECATTN_NAIVE_TOPP) {
        const int64_t B = va::naive_topp_batch_rows(R, N);
        w.skeys = reinterpret_cast<float*>(take((size_t)B * N * 4));
        w.vals_in = reinterpret_cast<int32_t*>(take((size_t)B * N * 4));
        w.vals_out = reinterpret_cast<int32_t*>(take((size_t)B * N * 4));
        w.seg_begin = reinterpret_cast<int64_t*>(take((size_t)B * 8));
        w.seg_end = reinterpret_cast<int64_t*>(take((size_t)B * 8));
        w.temp_bytes = va::naive_topp_sort_temp_bytes(B, N);
        w.temp = take(w.temp_bytes);
    }
    w.total = off;
    return w;
}
}  // namespace

size_t vecattn_select_naive_workspace_bytes(const vecattn_problem_t* p, int32_t pq, int32_t mode) {
    if (check_problem(p) != VECATTN_OK || (pq != 64 && pq != 128) ||
        (mode != VECATTN_NAIVE_MINS && mode != VECATTN_NAIVE_TOPP))
        return 0;
    return carve_select(p, pq, nullptr).total + carve_naive(p, pq, mode, nullptr).total + kAlign;
}

vecattn_status_t vecattn_select_naive(const vecattn_problem_t* p, int32_t pq, int32_t mode, float alpha, float top_p,
                                      const void* q, const void* k, int64_t* offsets, int32_t* indices, int64_t cap,
                                      int64_t* d_nnz, void* ws, size_t ws_bytes, vecattn_stream_t stream) {
    vecattn_status_t st = check_problem(p);
    if (st != VECATTN_OK) return st;
    if ((pq != 64 && pq != 128) || (mode != VECATTN_NAIVE_MINS && mode != VECATTN_NAIVE_TOPP) || !q || !k ||
        !offsets || !d_nnz || cap < 0 || (cap > 0 && !indices))
        return VECATTN_ERR_INVALID_ARGUMENT;
    if (mode == VECATTN_NAIVE_MINS && !(alpha >= 0.f && alpha < INFINITY)) return VECATTN_ERR_INVALID_ARGUMENT;
    if (mode == VECATTN_NAIVE_TOPP && !(top_p > 0.f && top_p <= 1.f)) return VECATTN_ERR_INVALID_ARGUMENT;
    if (!aligned16(q) || !aligned16(k)) return VECATTN_ERR_SHAPE;
    const size_t need = vecattn_select_naive_workspace_bytes(p, pq, mode);
    if (!ws || ws_bytes < need) return VECATTN_ERR_WORKSPACE;
    if (!aligned16(ws)) return VECATTN_ERR_SHAPE;
    cudaStream_t cs = (cudaStream_t)stream;
    const SelectWs w = carve_select(p, pq, ws);
    const NaiveWs nw = carve_naive(p, pq, mode, static_cast<uint8_t*>(ws) + w.total);
    vecattn_select_params_t s;
    memset(&s, 0, sizeof(s));
    s.mode = VECATTN_SEL_MINS_EXACT;
    s.pq = pq;
    s.bk = 16;
    s.gk = 1;
    s.alpha = alpha;
    SelectParams* sp = new SelectParams;
    st = fill_select_params(p, &s, pq, k, w, *sp);
    if (st == VECATTN_OK) st = set_k_map(p, k, 256, *sp);
    if (st != VECATTN_OK) { delete sp; return st; }
    sp->scores_out = nw.scores;
    plan_segments(p, &s, va::EPI_SCORES, *sp);
    const float scale = eff_scale(p);
    const float alpha_raw = sp->alpha_raw[0];  // alpha / scale, exactly as the fused MINS_EXACT
    const int64_t R = sp->BH * sp->Np;
    if (g_timing.enabled) {
        tbegin(true, true);
        g_timing.has_attn = false;
    }
    tmark(0, cs);
    cudaError_t e = va::launch_pool(q, w.qp, sp->BH, p->N, p->D, pq, cs);
    if (e == cudaSuccess) e = va::launch_select(*sp, va::EPI_SCORES, (int)p->D, cs);  // S_p -> HBM
    tmark(1, cs);
    const float sl2 = scale * 1.4426950408889634f;
    if (e == cudaSuccess)
        e = va::launch_naive_row_stats(nw.scores, R, sp->Np, p->N, pq, p->causal ? 1 : 0, sl2,
                                       mode == VECATTN_NAIVE_TOPP ? 1 : 0, nw.rmax, nw.rz, cs);
    if (e == cudaSuccess) {
        if (mode == VECATTN_NAIVE_MINS)
            e = va::launch_naive_mins(nw.scores, R, sp->Np, p->N, pq, p->causal ? 1 : 0, nw.rmax, alpha_raw, w.bitmask,
                                      sp->words_per_row, w.counts, cs);
        else
            e = va::launch_naive_topp(nw.scores, R, sp->Np, p->N, pq, p->causal ? 1 : 0, sl2, top_p, nw.rmax, nw.rz,
                                      nw.skeys, nw.vals_in, nw.vals_out, nw.seg_begin, nw.seg_end, nw.temp,
                                      nw.temp_bytes, w.bitmask, sp->words_per_row, w.counts, cs);
    }
    if (e == cudaSuccess) e = va::launch_scan(w.counts, R, offsets, d_nnz, cs);
    if (e == cudaSuccess && indices && cap > 0)
        e = va::launch_emit(w.bitmask, sp->words_per_row, offsets, d_nnz, cap, indices, sp->BH, sp->Np, p->N, pq,
                            p->causal ? 1 : 0, cs);
    tmark(2, cs);
    tmark(3, cs);
    delete sp;
    return cuda_status(e);
}


const char* vecattn_last_cuda_error(void) { return cudaGetErrorString(g_last_cuda_error); }

const char* vecattn_status_string(vecattn_status_t s) {
    switch (s) {
        case VECATTN_OK: return "ok";
        case VECATTN_ERR_INVALID_ARGUMENT: return "invalid argument";
        case VECATTN_ERR_SHAPE: return "unsupported or invalid shape";
        case VECATTN_ERR_UNSUPPORTED: return "unsupported device or driver";
        case VECATTN_ERR_WORKSPACE: return "workspace too small";
        case VECATTN_ERR_CUDA: return "CUDA launch error";
    }
    return "unknown status";
}

vecattn_status_t vecattn_pool(const vecattn_problem_t* p, int32_t pq, const void* q, void* qp,
                              vecattn_stream_t stream) {
    vecattn_status_t st = check_problem(p);
    if (st != VECATTN_OK) return st;
    if (pq != 64 && pq != 128) return VECATTN_ERR_INVALID_ARGUMENT;
    if (!q || !qp) return VECATTN_ERR_INVALID_ARGUMENT;
    if (!aligned16(q) || !aligned16(qp)) return VECATTN_ERR_SHAPE;
    VA_CU(va::launch_pool(q, qp, p->B * p->Hq, p->N, p->D, pq, (cudaStream_t)stream));
    return VECATTN_OK;
}

size_t vecattn_select_workspace_bytes(const vecattn_problem_t* p, const vecattn_select_params_t* s) {
    if (check_problem(p) != VECATTN_OK || !s || (s->pq != 64 && s->pq != 128)) return 0;
    return carve_select(p, s->pq, nullptr, s->mode == VECATTN_SEL_TOPK).total;
}

vecattn_status_t vecattn_select(const vecattn_problem_t* p, const vecattn_select_params_t* s, const void* q,
                                const void* k, int64_t* offsets, int32_t* indices, int64_t cap, int64_t* d_nnz,
                                void* ws, size_t ws_bytes, vecattn_stream_t stream) {
    vecattn_status_t st = check_select(p, s);
    if (st != VECATTN_OK) return st;
    if (!q || !k || !offsets || !d_nnz || cap < 0 || (cap > 0 && !indices)) return VECATTN_ERR_INVALID_ARGUMENT;
    if (!aligned16(q) || !aligned16(k)) return VECATTN_ERR_SHAPE;
    const SelectWs need = carve_select(p, s->pq, nullptr, s->mode == VECATTN_SEL_TOPK);
    if (!ws || ws_bytes < need.total) return VECATTN_ERR_WORKSPACE;
    if (!aligned16(ws)) return VECATTN_ERR_SHAPE;
    cudaStream_t cs = (cudaStream_t)stream;
    const SelectWs w = carve_select(p, s->pq, ws, s->mode == VECATTN_SEL_TOPK);
    SelectParams* sp = new SelectParams;
    st = fill_select_params(p, s, s->pq, k, w, *sp);
    if (st != VECATTN_OK) { delete sp; return st; }
    cudaError_t e = run_select(p, s, q, k, offsets, d_nnz, w, *sp, cs);
    if (e == cudaSuccess && indices && cap > 0)
        e = va::launch_emit(w.bitmask, sp->words_per_row, offsets, d_nnz, cap, indices, sp->BH, sp->Np, p->N,
                            s->pq, p->causal ? 1 : 0, cs);
    delete sp;
    return cuda_status(e);
}

vecattn_status_t vecattn_debug_scores(const vecattn_problem_t* p, int32_t pq, const void* q, const void* k,
                                      float* scores, void* ws, size_t ws_bytes, vecattn_stream_t stream) {
    vecattn_status_t st = check_problem(p);
    if (st != VECATTN_OK) return st;
    if ((pq != 64 && pq != 128) || !q || !k || !scores) return VECATTN_ERR_INVALID_ARGUMENT;
    const SelectWs need = carve_select(p, pq, nullptr);
    if (!ws || ws_bytes < need.total) return VECATTN_ERR_WORKSPACE;
    cudaStream_t cs = (cudaStream_t)stream;
    const SelectWs w = carve_select(p, pq, ws);
    vecattn_select_params_t s;
    memset(&s, 0, sizeof(s));
    s.pq = pq;
    s.bk = 16;
    s.gk = 1;
    SelectParams* sp = new SelectParams;
    st = fill_select_params(p, &s, pq, k, w, *sp);
    if (st == VECATTN_OK) st = set_k_map(p, k, 256, *sp);
    if (st != VECATTN_OK) { delete sp; return st; }
    sp->scores_out = scores;
    plan_segments(p, &s, va::EPI_SCORES, *sp);
    cudaError_t e = va::launch_pool(q, w.qp, sp->BH, p->N, p->D, pq, cs);
    if (e == cudaSuccess) e = va::launch_select(*sp, va::EPI_SCORES, (int)p->D, cs);
    delete sp;
    return cuda_status(e);
}

// Longest-first item order within each head (non-causal plans): the dynamic
// scheduler hands out a head's largest items first, so the step ends on its smallest ones.
// VECATTN_ITEM_ORDER=0 keeps the position order (A/B knob).
// Work window (vecattn_replica_t item_begin/item_end): only items [lo, hi) of the flattened
// bh * n_mt + it order are scheduled, always through an order array.
static cudaError_t item_order(AttnParams& ap, int32_t* order, cudaStream_t cs, int64_t lo, int64_t hi) {
    static const int mode = [] {  // 0 position order, 1 non-causal only (default), 2 causal too
        const char* e = getenv("VECATTN_ITEM_ORDER");
        return e == nullptr ? 1 : atoi(e);
    }();
    const bool windowed = lo != 0 || hi != ap.BH * ap.n_mt;
    ap.item_order = nullptr;
    ap.total_items = hi - lo;
    if (!windowed && ((ap.causal && mode < 2) || mode == 0 || ap.n_mt > va::kLptMaxItems)) return cudaSuccess;
    ap.item_order = order;
    if (windowed) ap.die_mode = 0;  // the per-die scheduler walks whole heads
    const int32_t by_position = mode == 0 || (ap.causal && mode < 2) ? 1 : 0;
    return va::launch_lpt_order(ap.wl_len, ap.BH, ap.n_mt, lo, hi, by_position, order, cs);
}

size_t vecattn_sparse_workspace_bytes(const vecattn_problem_t* p, int32_t pq, int64_t nnz_cap) {
    if (check_problem(p) != VECATTN_OK || (pq != 64 && pq != 128) || nnz_cap < 0) return 0;
    const int64_t n_it = (p->N + 255) / 256;
    return align_up((size_t)nnz_cap * 4) + align_up((size_t)(p->B * p->Hq * n_it) * 12) +
           align_up((size_t)(p->B * p->Hq * n_it) * 4) + kAlign;
}

// Attention workspace: plan entries [nnz_cap], segment lengths [items][3], item order
// [items] (per-head longest-first, non-causal), scheduler counters.
struct AttnWs {
    uint32_t* wl;
    int32_t* wl_len;
    int32_t* order;
    int* counter;
};
static AttnWs carve_attn(uint8_t* b, int64_t nnz_cap, int64_t items) {
    AttnWs w;
    w.wl = reinterpret_cast<uint32_t*>(b);
    b += align_up((size_t)nnz_cap * 4);
    w.wl_len = reinterpret_cast<int32_t*>(b);
    b += align_up((size_t)items * 12);
    w.order = reinterpret_cast<int32_t*>(b);
    b += align_up((size_t)items * 4);
    w.counter = reinterpret_cast<int*>(b);
    return w;
}

static vecattn_status_t attn_common(const vecattn_problem_t* p, const void* q, const void* k, const void* v,
                                    void* o, float* lse, AttnParams& ap) {
    memset(&ap, 0, sizeof(ap));
    const float scale = eff_scale(p);
    ap.q = (const __nv_bfloat16*)q;
    ap.k = (const __nv_bfloat16*)k;
    ap.v = (const __nv_bfloat16*)v;
    ap.o = (__nv_bfloat16*)o;
    ap.lse = lse;
    ap.N = p->N;
    ap.BH = p->B * p->Hq;
    ap.Hq = p->Hq;
    ap.Hkv = p->Hkv;
    ap.n_mt = (p->N + 255) / 256;
    ap.total_items = ap.BH * ap.n_mt;
    ap.causal = p->causal ? 1 : 0;
    ap.scale = scale;
    ap.scale_log2 = scale * 1.4426950408889634f;
    {
        const char* dm = getenv("VECATTN_DIE_SPLIT");
        ap.die_mode = dm ? atoi(dm) : 0;
        ap.strict_sync = getenv("VECATTN_STRICT_SYNC") ? 1 : 0;
    }
    {   // debug timeline: VECATTN_TRACE=<device pointer as decimal> (tests/scripts only)
        const char* tr = getenv("VECATTN_TRACE");
        ap.trace = tr ? reinterpret_cast<long long*>(strtoull(tr, nullptr, 10)) : nullptr;
    }
    if (!tmap_3d(&ap.tm_q, q, (uint64_t)p->D, (uint64_t)p->N, (uint64_t)ap.BH, 128)) return VECATTN_ERR_UNSUPPORTED;
    return VECATTN_OK;
}

static int attn_grid(int64_t items) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(items, va::grid_sms()));
}

vecattn_status_t vecattn_sparse_fwd(const vecattn_problem_t* p, int32_t pq, const void* q, const void* k,
                                    const void* v, const int64_t* offsets, const int32_t* indices, int64_t nnz_cap,
                                    void* o, float* lse, void* ws, size_t ws_bytes, vecattn_stream_t stream) {
    vecattn_status_t st = check_problem(p);
    if (st != VECATTN_OK) return st;
    if ((pq != 64 && pq != 128) || !q || !k || !v || !offsets || !o || nnz_cap < 0 || (nnz_cap > 0 && !indices))
        return VECATTN_ERR_INVALID_ARGUMENT;
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o)) return VECATTN_ERR_SHAPE;
    const size_t need = vecattn_sparse_workspace_bytes(p, pq, nnz_cap);
    if (!ws || ws_bytes < need) return VECATTN_ERR_WORKSPACE;
    cudaStream_t cs = (cudaStream_t)stream;
    AttnParams* ap = new AttnParams;
    st = attn_common(p, q, k, v, o, lse, *ap);
    const int64_t rows_kv = p->B * p->Hkv * p->N;
    if (st == VECATTN_OK && (!tmap_gather(&ap->tm_k, k, (uint64_t)p->D, (uint64_t)rows_kv) ||
                             !tmap_gather(&ap->tm_v, v, (uint64_t)p->D, (uint64_t)rows_kv)))
        st = VECATTN_ERR_UNSUPPORTED;
    if (st != VECATTN_OK) { delete ap; return st; }
    const AttnWs aw = carve_attn(static_cast<uint8_t*>(ws), nnz_cap, ap->BH * ap->n_mt);
    uint32_t* wl = aw.wl;
    int32_t* wl_len = aw.wl_len;
    int* counter = aw.counter;
    ap->Np = n_pooled(p, pq);
    ap->pq = pq;
    ap->wl = wl;
    ap->offsets = offsets;
    ap->wl_len = wl_len;
    ap->work_counter = counter;
    // capacity guard: nnz = offsets[R] beyond the plan's nnz_cap skips the plan and
    // the attention on the device instead of writing past the workspace
    ap->d_nnz = offsets + ap->BH * ap->Np;
    ap->nnz_cap = nnz_cap;
    if (g_timing.enabled) tbegin(false, true);
    tmark(1, cs);
    cudaError_t e = va::launch_worklist(offsets, indices ? indices : reinterpret_cast<const int32_t*>(wl), wl, wl_len,
                                        ap->BH, ap->Np, ap->n_mt, p->N, pq, nnz_cap, cs);
    if (e == cudaSuccess) e = item_order(*ap, aw.order, cs, 0, ap->BH * ap->n_mt);
    if (e == cudaSuccess) e = cudaMemsetAsync(counter, 0, 2 * sizeof(int), cs);
    tmark(2, cs);
    if (e == cudaSuccess) e = va::launch_attn(*ap, (int)p->D, true, attn_grid(ap->total_items), cs);
    tmark(3, cs);
    delete ap;
    return cuda_status(e);
}

size_t vecattn_dense_workspace_bytes(const vecattn_problem_t* p) {
    if (check_problem(p) != VECATTN_OK) return 0;
    return kAlign;
}

vecattn_status_t vecattn_dense_fwd(const vecattn_problem_t* p, const void* q, const void* k, const void* v, void* o,
                                   float* lse, void* ws, size_t ws_bytes, vecattn_stream_t stream) {
    vecattn_status_t st = check_problem(p);
    if (st != VECATTN_OK) return st;
    if (!q || !k || !v || !o) return VECATTN_ERR_INVALID_ARGUMENT;
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o)) return VECATTN_ERR_SHAPE;
    if (!ws || ws_bytes < kAlign) return VECATTN_ERR_WORKSPACE;
    cudaStream_t cs = (cudaStream_t)stream;
    AttnParams* ap = new AttnParams;
    st = attn_common(p, q, k, v, o, lse, *ap);
    if (st == VECATTN_OK &&
        (!tmap_3d(&ap->tm_k, k, (uint64_t)p->D, (uint64_t)p->N, (uint64_t)(p->B * p->Hkv), 128) ||
         !tmap_3d(&ap->tm_v, v, (uint64_t)p->D, (uint64_t)p->N, (uint64_t)(p->B * p->Hkv), 128)))
        st = VECATTN_ERR_UNSUPPORTED;
    if (st != VECATTN_OK) { delete ap; return st; }
    ap->Np = (p->N + 127) / 128;
    ap->pq = 128;
    ap->work_counter = reinterpret_cast<int*>(ws);
    cudaError_t e = cudaMemsetAsync(ws, 0, 2 * sizeof(int), cs);
    if (g_timing.enabled) tbegin(false, false);
    tmark(2, cs);
    if (e == cudaSuccess) e = va::launch_attn(*ap, (int)p->D, false, attn_grid(ap->total_items), cs);
    tmark(3, cs);
    delete ap;
    return cuda_status(e);
}

vecattn_status_t vecattn_validate_selection(const vecattn_problem_t* p, int32_t pq, const int64_t* offsets,
                                            const int32_t* indices, int32_t* d_bad, vecattn_stream_t stream) {
    vecattn_status_t st = check_problem(p);
    if (st != VECATTN_OK) return st;
    if ((pq != 64 && pq != 128) || !offsets || !d_bad) return VECATTN_ERR_INVALID_ARGUMENT;
    cudaStream_t cs = (cudaStream_t)stream;
    const int64_t Np = n_pooled(p, pq), R = p->B * p->Hq * Np;
    VA_CU(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), cs));
    validate_kernel<<<(unsigned)((R + 255) / 256), 256, 0, cs>>>(offsets, indices, R, Np, p->N, pq,
                                                                  p->causal ? 1 : 0, d_bad);
    VA_CU(cudaGetLastError());
    return VECATTN_OK;
}


size_t vecattn_forward_workspace_bytes(const vecattn_problem_t* p, const vecattn_select_params_t* s,
                                       int64_t nnz_cap) {
    if (check_problem(p) != VECATTN_OK || !s || (s->pq != 64 && s->pq != 128) || nnz_cap < 0) return 0;
    return carve_select(p, s->pq, nullptr, s->mode == VECATTN_SEL_TOPK).total + vecattn_sparse_workspace_bytes(p, s->pq, nnz_cap);
}

static vecattn_status_t forward_impl(const vecattn_problem_t* p, const vecattn_select_params_t* s, const void* q,
                                     const void* k, const void* v, int64_t* offsets, int32_t* indices, int64_t cap,
                                     int64_t* d_nnz, int64_t nnz_cap, void* o, float* lse,
                                     const vecattn_replica_t* rep, void* ws, size_t ws_bytes,
                                     vecattn_stream_t stream) {
    vecattn_status_t st = check_select(p, s);
    if (st != VECATTN_OK) return st;
    const bool replicate = rep != nullptr && (rep->n_peers > 0 || rep->o_multicast != nullptr);
    if (!q || !k || !v || (!o && !replicate) || !offsets || !d_nnz || cap < 0 || (cap > 0 && !indices) ||
        nnz_cap < 0)
        return VECATTN_ERR_INVALID_ARGUMENT;
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || (o && !aligned16(o))) return VECATTN_ERR_SHAPE;
    if (rep != nullptr) {
        if (rep->n_peers < 0 || rep->n_peers > 8 || rep->head0 < 0 || rep->head0 + p->Hq > rep->heads_total)
            return VECATTN_ERR_INVALID_ARGUMENT;
        const int64_t n_items = p->B * p->Hq * ((p->N + 255) / 256);
        if (rep->item_end > 0 && (rep->item_begin < 0 || rep->item_begin >= rep->item_end || rep->item_end > n_items))
            return VECATTN_ERR_INVALID_ARGUMENT;
        for (int i = 0; i < rep->n_peers && rep->o_multicast == nullptr; ++i) {
            if (!rep->peer_o[i]) return VECATTN_ERR_INVALID_ARGUMENT;
            if (!aligned16(rep->peer_o[i])) return VECATTN_ERR_SHAPE;
        }
        if (rep->o_multicast && !aligned16(rep->o_multicast)) return VECATTN_ERR_SHAPE;
    }
    const size_t need = vecattn_forward_workspace_bytes(p, s, nnz_cap);
    if (!ws || ws_bytes < need) return VECATTN_ERR_WORKSPACE;
    if (!aligned16(ws)) return VECATTN_ERR_SHAPE;
    cudaStream_t cs = (cudaStream_t)stream;
    const SelectWs w = carve_select(p, s->pq, ws, s->mode == VECATTN_SEL_TOPK);
    uint8_t* b = static_cast<uint8_t*>(ws) + w.total;
    SelectParams* sp = new SelectParams;
    AttnParams* ap = new AttnParams;
    st = fill_select_params(p, s, s->pq, k, w, *sp);
    if (st == VECATTN_OK) st = attn_common(p, q, k, v, o, lse, *ap);
    const int64_t rows_kv = p->B * p->Hkv * p->N;
    if (st == VECATTN_OK && (!tmap_gather(&ap->tm_k, k, (uint64_t)p->D, (uint64_t)rows_kv) ||
                             !tmap_gather(&ap->tm_v, v, (uint64_t)p->D, (uint64_t)rows_kv)))
        st = VECATTN_ERR_UNSUPPORTED;
    if (st != VECATTN_OK) { delete sp; delete ap; return st; }
    const int64_t n_items = ap->BH * ap->n_mt;
    int64_t win_lo = 0, win_hi = n_items;
    if (rep != nullptr && rep->item_end > 0) {
        win_lo = rep->item_begin;
        win_hi = rep->item_end;
    }
    if (replicate) {
        ap->o_mc = static_cast<__nv_bfloat16*>(rep->o_multicast);
        ap->rep_n = rep->o_multicast ? 0 : rep->n_peers;
        for (int i = 0; i < ap->rep_n; ++i) ap->rep_o[i] = static_cast<__nv_bfloat16*>(rep->peer_o[i]);
        ap->rep_head0 = rep->head0;
        ap->rep_heads = rep->heads_total;
    }
    const AttnWs aw = carve_attn(b, nnz_cap, ap->BH * ap->n_mt);
    uint32_t* wl = aw.wl;
    int32_t* wl_len = aw.wl_len;
    int* counter = aw.counter;
    ap->Np = sp->Np;
    ap->pq = s->pq;
    ap->wl = wl;
    ap->offsets = offsets;
    ap->wl_len = wl_len;
    ap->work_counter = counter;
    ap->d_nnz = d_nnz;
    ap->nnz_cap = nnz_cap;
    if (g_timing.enabled) tbegin(true, true);
    // The CSR (the caller's index lists) is not an input of the attention, which reads the
    // plan: by default it is emitted on a side stream beside the attention kernel (one small
    // CTA per SM next to the persistent attention CTA), forked after the plan and joined
    // before the call's work on `stream` ends.  VECATTN_SERIAL_EMIT=1 emits before the plan.
    const bool emit = indices && cap > 0;
    // (non-causal only: the causal attention kernel holds all 64K registers of its SM, so a
    // side CTA could not run beside it)
    // (a stream being captured into a CUDA graph keeps the serial order: the library-global
    // side stream must not be pulled into the caller's capture)
    cudaStreamCaptureStatus capst = cudaStreamCaptureStatusNone;
    const bool capturing = cudaStreamIsCapturing(cs, &capst) == cudaSuccess && capst != cudaStreamCaptureStatusNone;
    SideStream* side =
        (emit && !p->causal && !capturing && !getenv("VECATTN_SERIAL_EMIT") && !va::attn_uses_pair(*ap, (int)p->D, true))
            ? side_stream()
            : nullptr;
    tmark(0, cs);
    cudaError_t e = run_select(p, s, q, k, offsets, d_nnz, w, *sp, cs);
    tmark(1, cs);
    if (e == cudaSuccess && emit && !side)
        e = va::launch_emit(w.bitmask, sp->words_per_row, offsets, d_nnz, cap, indices, sp->BH, sp->Np, p->N, s->pq,
                            p->causal ? 1 : 0, cs);
    if (e == cudaSuccess)
        e = va::launch_plan(w.bitmask, sp->words_per_row, offsets, d_nnz, nnz_cap, wl, wl_len, sp->BH, sp->Np, p->N,
                            s->pq, p->causal ? 1 : 0, cs);
    if (e == cudaSuccess) e = item_order(*ap, aw.order, cs, win_lo, win_hi);
    if (e == cudaSuccess) e = cudaMemsetAsync(counter, 0, 2 * sizeof(int), cs);
    tmark(2, cs);
    std::unique_lock<std::mutex> lk;
    if (e == cudaSuccess && side) {
        lk = std::unique_lock<std::mutex>(side->mu);
        e = cudaEventRecord(side->ev_fork, cs);
    }
    if (e == cudaSuccess) e = va::launch_attn(*ap, (int)p->D, true, attn_grid(ap->total_items), cs);
    tmark(3, cs);
    if (e == cudaSuccess && side) {
        e = cudaStreamWaitEvent(side->s, side->ev_fork, 0);
        if (e == cudaSuccess)
            e = va::launch_emit_shadow(w.bitmask, sp->words_per_row, offsets, d_nnz, cap, indices, sp->BH, sp->Np,
                                       p->N, s->pq, p->causal ? 1 : 0, side->sms, side->s);
        if (e == cudaSuccess) e = cudaEventRecord(side->ev_join, side->s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, side->ev_join, 0);
    }
    delete sp;
    delete ap;
    return cuda_status(e);
}

vecattn_status_t vecattn_forward(const vecattn_problem_t* p, const vecattn_select_params_t* s, const void* q,
                                 const void* k, const void* v, int64_t* offsets, int32_t* indices, int64_t cap,
                                 int64_t* d_nnz, int64_t nnz_cap, void* o, float* lse, void* ws, size_t ws_bytes,
                                 vecattn_stream_t stream) {
    return forward_impl(p, s, q, k, v, offsets, indices, cap, d_nnz, nnz_cap, o, lse, nullptr, ws, ws_bytes, stream);
}

vecattn_status_t vecattn_forward_replicated(const vecattn_problem_t* p, const vecattn_select_params_t* s,
                                            const void* q, const void* k, const void* v, int64_t* offsets,
                                            int32_t* indices, int64_t cap, int64_t* d_nnz, int64_t nnz_cap, void* o,
                                            float* lse, const vecattn_replica_t* rep, void* ws, size_t ws_bytes,
                                            vecattn_stream_t stream) {
    return forward_impl(p, s, q, k, v, offsets, indices, cap, d_nnz, nnz_cap, o, lse, rep, ws, ws_bytes, stream);
}

}  // extern "C"
