// vecattn_oracle.cpp — plain, slow, fp64 CPU ORACLE for VecAttention (arXiv 2603.29494).
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  The product path
// (paper_2603_29494_b200/) never links, imports or calls it, and this file shares
// no code, header, table or constant with paper_2603_29494_b200/csrc/.
//
// Every function works on ONE attention head with row-major fp64 arrays (the
// caller up-converts the exact bf16 bit patterns the GPU sees; bf16 -> fp64 is
// exact).  Loops follow the paper's definitions in its own order; the only
// parallelism is an OpenMP loop over independent output rows.
//
// Citations: P:<line> = /root/reference/PAPER.md line, S:<line> = SPEC.md line.
//   Eq. 1 dense attention ............ P:54-68 (Sec. 2.1)
//   Eq. 2 query pooling ............... P:187-194 (Sec. 3.1.1), Alg. 1 line P:770
//   Eq. 3 minS filter ................. P:218-232 (Sec. 3.1.2)
//   topP naive filter ................. P:203-216 (Sec. 3.1.1-3.1.2)
//   TilingSelect / G_K running max .... P:268-278, P:290-307 (Sec. 3.1.3)
//   Alg. 1 important-vector selection . P:755-850 (App. D.1)
//   Eq. 5 vector-sparse attention ..... P:309-341 (Sec. 3.2), Alg. 2
// Readings of ambiguous passages are the ones listed in DESIGN.md "Readings"
// (R1..R14); each use below names its reading.
//
// Parity pins: see tests/test_oracle_*.py (closed forms, worked examples,
// brute force, torch fp64 SDPA, invariants).

#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <limits>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

const double NEG_INF = -std::numeric_limits<double>::infinity();

// Round a double to the nearest bfloat16 value, ties to even (IEEE RNE), by the
// definition: x = r * 2^(e-8) with r an integer of at most 8 significant bits.
// bf16 = 1 sign, 8 exponent (bias 127), 7 stored mantissa bits; smallest
// subnormal 2^-133.  Returns the rounded value as a double (exactly
// representable).  Reading R11: Q_p is RNE-bf16 of the exact mean.
double bf16_rne(double x) {
    if (x == 0.0 || !std::isfinite(x)) return x;
    int e;                                   // x = m * 2^e, 0.5 <= |m| < 1
    std::frexp(x, &e);
    int q = e - 8;                           // quantum exponent for 8 significant bits
    if (q < -133) q = -133;                  // subnormal range: fixed quantum 2^-133
    double scaled = std::ldexp(x, -q);       // exact (power-of-two scaling)
    double r = std::nearbyint(scaled);       // default rounding mode: nearest, ties to even
    return std::ldexp(r, q);                 // overflow to inf is not reachable for our inputs
}

// Eq. 2: Q_p[i] = (1/h_i) * sum_{t in block i} Q[t];
// ragged last block uses its true height h_i (reading R7).
void pool_rows(const double* q, int64_t N, int64_t D, int32_t pq, int32_t round_bf16,
               double* qp) {
    const int64_t Np = (N + pq - 1) / pq;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < Np; ++i) {
        const int64_t r0 = i * pq;
        const int64_t r1 = std::min<int64_t>(N, r0 + pq);
        const double h = double(r1 - r0);
        for (int64_t d = 0; d < D; ++d) {
            double s = 0.0;
            for (int64_t r = r0; r < r1; ++r) s += q[r * D + d];
            double mean = s / h;
            qp[i * D + d] = round_bf16 ? bf16_rne(mean) : mean;
        }
    }
}

double dot(const double* a, const double* b, int64_t D) {
    double s = 0.0;
    for (int64_t d = 0; d < D; ++d) s += a[d] * b[d];
    return s;
}

// Visible key range of pooled row i: all of [0,N) non-causal; [0, L_i] causal with
// L_i = min(N,(i+1)P_q) - 1, the block's LAST query row (reading R5).
int64_t visible_end(int64_t i, int64_t N, int32_t pq, int32_t causal) {
    if (!causal) return N;
    return std::min<int64_t>(N, (i + 1) * (int64_t)pq);
}

}  // namespace

extern "C" {

int oracle_version() { return 1; }

int oracle_num_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

// Element-wise RNE rounding of doubles to bf16 values (returned as doubles).
void oracle_round_bf16(const double* x, int64_t n, double* out) {
    for (int64_t t = 0; t < n; ++t) out[t] = bf16_rne(x[t]);
}

// Eq. 2 for one head. q: [N,D]; qp: [ceil(N/pq), D].
int oracle_pool(const double* q, int64_t N, int64_t D, int32_t pq, int32_t round_bf16,
                double* qp) {
    if (!q || !qp || N < 1 || D < 1 || pq < 1) return 1;
    pool_rows(q, N, D, pq, round_bf16, qp);
    return 0;
}

// Pooled scores s_ij = scale * <Q_p[i], k_j> for one row.
int oracle_scores_row(const double* qp, const double* k, int64_t N, int64_t D, double scale,
                      int64_t i, double* s_out) {
    const double* a = qp + i * D;
    for (int64_t j = 0; j < N; ++j) s_out[j] = scale * dot(a, k + j * D, D);
    return 0;
}

// Important-vector selection for a list of pooled rows of ONE head.
//   mode 0 = MINS_ALG1  : Alg. 1 literally: per group of G_K tiles of
//                          B_K keys reset m = -inf (listing P:796, reading R2); per tile
//                          in ascending order m = max(m, rowmax(tile)) THEN keep
//                          s >= m - alpha (reading R3; '>=' of Eq. 3, R1).
//   mode 1 = MINS_EXACT : Eq. 3 with m = max over all visible keys.
//   mode 2 = TOPK       : the k_i largest, ties -> lowest index (R12);
//                          k_i = min(topk, |V_i|) if topk > 0 else
//                          clamp(floor(keep_frac*|V_i| + 0.5), 1, |V_i|).
// Causal: keys j > L_i excluded before max and filter (R5).
// Outputs per requested row r (pooled row rows[r]): counts[r] and ascending unique
// indices in idx[r*idx_stride ...] (capacity >= N).  Optional diagnostics:
//   thr[r*n_tiles + t]   threshold theta in force for B_K-tile t (ALG1: m_run - alpha;
//                        EXACT: m - alpha; TOPK: k-th largest score), NaN if tile invisible
//   jstar[r*n_tiles + t] key index that defines theta's m (argmax / k-th element)
// where n_tiles = ceil(N / bk).  Returns 0 on success, 1 on bad arguments.
int oracle_select_rows(const double* qp, const double* k, int64_t N, int64_t D, int32_t pq,
                       int32_t causal, double scale, int32_t mode, int32_t bk, int32_t gk,
                       double alpha, int64_t topk, double keep_frac,
                       const int64_t* rows, int64_t nrows,
                       int64_t* counts, int32_t* idx, int64_t idx_stride,
                       double* thr, int64_t* jstar) {
    if (!qp || !k || !rows || !counts || !idx || N < 1 || D < 1 || pq < 1 || bk < 1 ||
        gk < 1 || !(alpha >= 0.0) || idx_stride < N)
        return 1;
    if (mode == 2 && topk <= 0 && !(keep_frac > 0.0 && keep_frac <= 1.0)) return 1;
    const int64_t n_tiles = (N + bk - 1) / bk;
    const int64_t G = (int64_t)bk * (int64_t)gk;   // keys per group of G_K tiles

#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t i = rows[r];
        const int64_t vend = visible_end(i, N, pq, causal);   // visible keys: [0, vend)
        std::vector<double> s(vend);
        for (int64_t j = 0; j < vend; ++j) s[j] = scale * dot(qp + i * D, k + j * D, D);
        int32_t* out = idx + r * idx_stride;
        int64_t c = 0;
        double* th = thr ? thr + r * n_tiles : nullptr;
        int64_t* js = jstar ? jstar + r * n_tiles : nullptr;
        if (th) for (int64_t t = 0; t < n_tiles; ++t) th[t] = std::nan("");
        if (js) for (int64_t t = 0; t < n_tiles; ++t) js[t] = -1;

        if (mode == 0) {
            for (int64_t g0 = 0; g0 < N; g0 += G) {                 // i_g loop
                double m = NEG_INF;                                  // m_S <- -inf
                int64_t jm = -1;
                const int64_t gend = std::min<int64_t>(g0 + G, N);
                for (int64_t t0 = g0; t0 < gend; t0 += bk) {         // K-tile loop
                    const int64_t t1 = std::min<int64_t>(std::min<int64_t>(t0 + bk, gend), vend);
                    if (t1 <= t0) continue;                          // tile invisible (causal)
                    for (int64_t j = t0; j < t1; ++j)                // m_S <- max(m_S, rowmax)
                        if (s[j] > m) { m = s[j]; jm = j; }
                    const double theta = m - alpha;
                    for (int64_t j = t0; j < t1; ++j)                // M <- S >= m_S - alpha (R1)
                        if (s[j] >= theta) out[c++] = (int32_t)j;    // Indexing + Concatenate
                    if (th) th[t0 / bk] = theta;
                    if (js) js[t0 / bk] = jm;
                }
            }
        } else if (mode == 1) {
            double m = NEG_INF;
            int64_t jm = -1;
            for (int64_t j = 0; j < vend; ++j)                       // m_i^s = rowmax(s_i)
                if (s[j] > m) { m = s[j]; jm = j; }
            const double theta = m - alpha;
            for (int64_t j = 0; j < vend; ++j)                       // Eq. 3
                if (s[j] >= theta) out[c++] = (int32_t)j;
            if (th) for (int64_t t = 0; t * bk < vend; ++t) th[t] = theta;
            if (js) for (int64_t t = 0; t * bk < vend; ++t) js[t] = jm;
        } else {
            int64_t ki;
            if (topk > 0) ki = std::min<int64_t>(topk, vend);
            else {
                ki = (int64_t)std::floor(keep_frac * (double)vend + 0.5);
                ki = std::max<int64_t>(1, std::min<int64_t>(ki, vend));
            }
            std::vector<int64_t> order(vend);
            for (int64_t j = 0; j < vend; ++j) order[j] = j;
            std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
                if (s[a] != s[b]) return s[a] > s[b];
                return a < b;                                        // ties -> lowest index (R12)
            });
            std::vector<int32_t> sel(order.begin(), order.begin() + ki);
            std::sort(sel.begin(), sel.end());
            for (int64_t t = 0; t < ki; ++t) out[c++] = sel[t];
            const int64_t kth = order[ki - 1];
            if (th) for (int64_t t = 0; t * bk < vend; ++t) th[t] = s[kth];
            if (js) for (int64_t t = 0; t * bk < vend; ++t) js[t] = kth;
        }
        if (mode == 0) std::sort(out, out + c);   // already ascending; canonical form (R9)
        counts[r] = c;
    }
    return 0;
}

// topP ("nucleus") selection of the NAIVE approach: the estimated
// attention map A_p[i,:] = softmax_j(s_ij) over the visible keys (softmax of
// Eq. 1 applied to the pooled scores), then the smallest prefix of keys sorted by
// descending probability (ties -> lowest index, reading R12) whose cumulative mass is
// >= p; keys of zero probability (fp64 underflow) are never taken, so p >= 1 returns
// every nonzero-probability key.  Causal: keys j > L_i are excluded first (R5).
// Outputs per requested row r: counts[r], ascending indices in idx[r*idx_stride ...],
// and optionally mass[r] = the selected cumulative probability.  Returns 0 / 1 (bad args).
int oracle_topp_rows(const double* qp, const double* k, int64_t N, int64_t D, int32_t pq,
                     int32_t causal, double scale, double p, const int64_t* rows, int64_t nrows,
                     int64_t* counts, int32_t* idx, int64_t idx_stride, double* mass) {
    if (!qp || !k || !rows || !counts || !idx || N < 1 || D < 1 || pq < 1 || idx_stride < N ||
        !(p > 0.0 && p <= 1.0))
        return 1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t i = rows[r];
        const int64_t vend = visible_end(i, N, pq, causal);
        std::vector<double> s(vend), a(vend);
        for (int64_t j = 0; j < vend; ++j) s[j] = scale * dot(qp + i * D, k + j * D, D);
        double m = NEG_INF;                                          // softmax: max ...
        for (int64_t j = 0; j < vend; ++j) m = std::max(m, s[j]);
        double z = 0.0;                                              // ... normaliser ...
        for (int64_t j = 0; j < vend; ++j) z += std::exp(s[j] - m);
        for (int64_t j = 0; j < vend; ++j) a[j] = std::exp(s[j] - m) / z;   // ... A_p[i, j]
        std::vector<int64_t> order(vend);
        for (int64_t j = 0; j < vend; ++j) order[j] = j;
        std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
            if (a[x] != a[y]) return a[x] > a[y];                     // descending probability
            return x < y;                                            // ties -> lowest index (R12)
        });
        std::vector<int32_t> sel;
        double cum = 0.0;
        for (int64_t t = 0; t < vend; ++t) {                         // smallest prefix with mass >= p
            const int64_t j = order[t];
            if (a[j] == 0.0) break;                                  // zero probability: never taken
            sel.push_back((int32_t)j);
            cum += a[j];
            if (cum >= p) break;
        }
        std::sort(sel.begin(), sel.end());
        int32_t* out = idx + r * idx_stride;
        for (size_t t = 0; t < sel.size(); ++t) out[t] = sel[t];
        counts[r] = (int64_t)sel.size();
        if (mass) mass[r] = cum;
    }
    return 0;
}

// Eq. 5 for a list of query blocks of ONE head, written as the plain
// (non-online) softmax the online Alg. 2 reaches exactly.
//   blocks[b]     : query-block id i (rows [i*pq, min(N,(i+1)pq)))
//   sel_off/sel_idx: CSR over the requested blocks, sel_off[b]..sel_off[b+1] = Idx(i)
// Row r uses J_r = Idx(i) (non-causal, Alg. 2 mask = identity, R10) or
// {j in Idx(i): j <= r} (causal, Alg. 2 mask(S) P:911).  J_r empty -> O_r = V_r and
// LSE_r = scale*<q_r,k_r> (reading R6).
// o: [nblocks*pq, D] (rows past N left 0), lse: [nblocks*pq] (NaN past N).
int oracle_attn_blocks(const double* q, const double* k, const double* v, int64_t N, int64_t D,
                       int32_t pq, int32_t causal, double scale,
                       const int64_t* blocks, int64_t nblocks,
                       const int64_t* sel_off, const int32_t* sel_idx,
                       double* o, double* lse) {
    if (!q || !k || !v || !blocks || !sel_off || !o || N < 1 || D < 1 || pq < 1) return 1;
    for (int64_t b = 0; b < nblocks; ++b) {
        for (int64_t t = sel_off[b]; t < sel_off[b + 1]; ++t)
            if (sel_idx[t] < 0 || sel_idx[t] >= N) return 2;
    }
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
    for (int64_t b = 0; b < nblocks; ++b) {
        for (int64_t rr = 0; rr < pq; ++rr) {
            const int64_t i = blocks[b];
            const int64_t r = i * pq + rr;
            double* orow = o + (b * pq + rr) * D;
            if (r >= N) {
                for (int64_t d = 0; d < D; ++d) orow[d] = 0.0;
                if (lse) lse[b * pq + rr] = std::nan("");
                continue;
            }
            std::vector<int64_t> J;
            for (int64_t t = sel_off[b]; t < sel_off[b + 1]; ++t) {
                const int64_t j = sel_idx[t];
                if (!causal || j <= r) J.push_back(j);
            }
            if (J.empty()) {
                for (int64_t d = 0; d < D; ++d) orow[d] = v[r * D + d];
                if (lse) lse[b * pq + rr] = scale * dot(q + r * D, k + r * D, D);
                continue;
            }
            std::vector<double> x(J.size());
            double M = NEG_INF;
            for (size_t t = 0; t < J.size(); ++t) {
                x[t] = scale * dot(q + r * D, k + J[t] * D, D);
                M = std::max(M, x[t]);
            }
            double l = 0.0;
            for (size_t t = 0; t < J.size(); ++t) l += std::exp(x[t] - M);
            for (int64_t d = 0; d < D; ++d) orow[d] = 0.0;
            for (size_t t = 0; t < J.size(); ++t) {
                const double p = std::exp(x[t] - M);
                const double* vr = v + J[t] * D;
                for (int64_t d = 0; d < D; ++d) orow[d] += p * vr[d];
            }
            for (int64_t d = 0; d < D; ++d) orow[d] /= l;
            if (lse) lse[b * pq + rr] = M + std::log(l);
        }
    }
    return 0;
}

// Eq. 1 for a list of query rows of ONE head: S = scale*QK^T, causal
// entries j > r masked, A = softmax(S), O = AV, LSE = M + ln(l).
int oracle_dense_rows(const double* q, const double* k, const double* v, int64_t N, int64_t D,
                      int32_t causal, double scale, const int64_t* rows, int64_t nrows,
                      double* o, double* lse) {
    if (!q || !k || !v || !rows || !o || N < 1 || D < 1) return 1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < nrows; ++t) {
        const int64_t r = rows[t];
        const int64_t jend = causal ? r + 1 : N;
        std::vector<double> x(jend);
        double M = NEG_INF;
        for (int64_t j = 0; j < jend; ++j) {
            x[j] = scale * dot(q + r * D, k + j * D, D);
            M = std::max(M, x[j]);
        }
        double l = 0.0;
        for (int64_t j = 0; j < jend; ++j) l += std::exp(x[j] - M);
        double* orow = o + t * D;
        for (int64_t d = 0; d < D; ++d) orow[d] = 0.0;
        for (int64_t j = 0; j < jend; ++j) {
            const double p = std::exp(x[j] - M);
            for (int64_t d = 0; d < D; ++d) orow[d] += p * v[j * D + d];
        }
        for (int64_t d = 0; d < D; ++d) orow[d] /= l;
        if (lse) lse[t] = M + std::log(l);
    }
    return 0;
}

}  // extern "C"
