/* vecattn.h — C ABI of the B200 (sm_100a) VecAttention hot path.
 *
 * VecAttention (arXiv 2603.29494, /root/reference/PAPER.md = "P:<line>"):
 *   stage 1  important-vector selection: query pooling (Eq. 2) +
 *            TilingSelect with the minS filter (Eq. 3; Sec. 3.1.3
 *            P:268-307; Alg. 1) -> per-query-block sorted key indices;
 *   stage 2  vector-sparse attention (Eq. 5; Alg. 2);
 *   plus     dense attention (Eq. 1) as the in-library reference kernel.
 *
 * Conventions (all entry points):
 *  - Every tensor pointer is a DEVICE pointer (cudaMalloc / torch CUDA memory),
 *    16-byte aligned.  bf16 = IEEE bfloat16 bit patterns.  Layouts are dense,
 *    row-major:  Q [B, Hq, N, D],  K, V [B, Hkv, N, D],  O [B, Hq, N, D],
 *    LSE [B, Hq, N] fp32 (natural log).  GQA: query head h reads KV head
 *    h / (Hq / Hkv) (reading R13).
 *  - All work is enqueued asynchronously on `stream`; nothing is synchronised.
 *  - Ownership: the caller owns every buffer, including the workspace `ws`
 *    (size from the matching *_workspace_bytes()).  The library never allocates.
 *  - Errors: argument/shape problems return a status synchronously BEFORE any
 *    launch (no side effects).  Device faults surface at the caller's next sync as
 *    CUDA errors.  VECATTN_ERR_CUDA means a launch failed; cudaGetLastError() is
 *    left set.
 *  - Selection output is CSR over query blocks.  Row id r = (b*Hq + h)*N_p + i,
 *    N_p = ceil(N / pq).  offsets: int64 [B*Hq*N_p + 1], indices: int32 [nnz],
 *    ascending and unique within a row, each in [0, N), and <= L_i =
 *    min(N,(i+1)*pq)-1 when causal (reading R5).
 */
#ifndef VECATTN_H
#define VECATTN_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define VECATTN_API __attribute__((visibility("default")))
#else
#define VECATTN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* vecattn_stream_t; /* ABI-identical to cudaStream_t; NULL = legacy stream */

typedef enum {
    VECATTN_OK = 0,
    VECATTN_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, pq not in {64,128}, alpha < 0 or NaN, bk not in
                                         {8,...,256} (powers of 2), gk < 1, TOPK with neither topk > 0 nor
                                         keep_frac in (0,1], Hq % Hkv != 0, scale < 0 or NaN          */
    VECATTN_ERR_SHAPE = 2,            /* B, N < 1; D not in {64,128}; N >= 2^28; Hq > 1024; pointer not
                                         16-byte aligned; B*Hkv*N >= 2^31                              */
    VECATTN_ERR_UNSUPPORTED = 3,      /* no sm_100 device, or cuTensorMapEncodeTiled unavailable      */
    VECATTN_ERR_WORKSPACE = 4,        /* ws == NULL or ws_bytes < *_workspace_bytes()                 */
    VECATTN_ERR_CUDA = 5              /* a CUDA launch/API call failed                                */
} vecattn_status_t;

/* Problem statement (north_star: Q/K/V [B,H,N,d] bf16, causal flag). */
typedef struct {
    int64_t B, Hq, Hkv, N, D;
    int32_t causal;  /* 1 = VLM prefill (key j visible to query r iff j <= r); 0 = DiT     */
    float scale;     /* softmax scale tau; 0 => 1/sqrt(D) (Eq. 1; Alg. 2 line P:870) */
} vecattn_problem_t;

typedef enum {
    VECATTN_SEL_MINS_ALG1 = 0,  /* Alg. 1 exactly: running row max over B_K-key tiles, reset every
                                   G_K tiles, keep s >= m - alpha (readings R1-R3)          */
    VECATTN_SEL_MINS_EXACT = 1, /* Eq. 3 with the global row max (two GEMM passes)                  */
    VECATTN_SEL_TOPK = 2        /* per-block budget k_i, ties -> lowest index (R12)      */
} vecattn_sel_mode_t;

typedef struct {
    int32_t mode;                /* vecattn_sel_mode_t                                              */
    int32_t pq;                  /* vector size P_q = query-block size, 64 or 128   */
    int32_t bk;                  /* Alg. 1 K-tile size B_K: 8, 16, 32, 64, 128 or 256 (paper: 16)    */
    int32_t gk;                  /* Alg. 1 K-tiles per group G_K >= 1 (16 VLM, 8192 DiT)     */
    float alpha;                 /* minS filtering ratio (Eq. 3), >= 0, in scaled-logit units (R4)  */
    const float* alpha_per_head; /* HOST pointer [Hq] or NULL; overrides alpha per query head (Eq. 4) */
    int64_t topk;                /* TOPK: k_i = min(topk, |V_i|) when topk > 0, else ...             */
    float keep_frac;             /* ... k_i = clamp(floor(keep_frac*|V_i| + 0.5), 1, |V_i|)         */
} vecattn_select_params_t;

/* ---------------------------------------------------------------- stage 1 */

/* Eq. 2: qp [B,Hq,N_p,D] bf16 = RNE-bf16 of the exact fp64 block mean
 * (ragged last block: its true height, reading R7).  q, qp: device.              */
VECATTN_API vecattn_status_t vecattn_pool(const vecattn_problem_t* p, int32_t pq, const void* q, void* qp,
                              vecattn_stream_t stream);

VECATTN_API size_t vecattn_select_workspace_bytes(const vecattn_problem_t* p, const vecattn_select_params_t* s);

/* Important-vector selection (Alg. 1).  Writes `offsets` (always),
 * `*d_nnz` (device int64, always) and, iff indices != NULL and nnz <= cap, the
 * ascending `indices`.  Capacity protocol: if nnz > cap the contents of indices are
 * unspecified; read d_nnz, re-allocate and call again (indices = NULL, cap = 0 is a
 * counts-only call, e.g. for alpha calibration).  The estimated attention map is
 * never written to memory: scores live in TMEM, only a 1-bit mask per (block, key)
 * reaches HBM (workspace).                                                          */
VECATTN_API vecattn_status_t vecattn_select(const vecattn_problem_t* p, const vecattn_select_params_t* s,
                                const void* q, const void* k, int64_t* offsets, int32_t* indices,
                                int64_t cap, int64_t* d_nnz, void* ws, size_t ws_bytes,
                                vecattn_stream_t stream);

/* ---------------------------------------------------------------- stage 2 */

VECATTN_API size_t vecattn_sparse_workspace_bytes(const vecattn_problem_t* p, int32_t pq, int64_t nnz_cap);

/* Vector-sparse attention, Eq. 5 / Alg. 2: for every query
 * block i, O[rows of i] = softmax(scale * Q[rows] K[Idx(i)]^T) V[Idx(i)], causal rows
 * additionally masked to keys j <= r.  A row with no visible selected key outputs
 * O_r = V_r and LSE_r = scale*<q_r,k_r> (reading R6).  offsets/indices: CSR as
 * produced by vecattn_select (same pq); nnz = offsets[last] must be <= nnz_cap (the
 * workspace's plan capacity): if it is larger, the device skips the plan and the attention
 * (o/lse untouched) instead of writing past the workspace.
 * Index content is NOT validated (O(nnz)); out-of-range indices are undefined
 * behaviour -- see vecattn_validate_selection.  lse may be NULL.                    */
VECATTN_API vecattn_status_t vecattn_sparse_fwd(const vecattn_problem_t* p, int32_t pq, const void* q, const void* k,
                                    const void* v, const int64_t* offsets, const int32_t* indices,
                                    int64_t nnz_cap, void* o, float* lse, void* ws, size_t ws_bytes,
                                    vecattn_stream_t stream);

/* ------------------------------------------------------- fused stage 1+2 */

VECATTN_API size_t vecattn_forward_workspace_bytes(const vecattn_problem_t* p, const vecattn_select_params_t* s,
                                                   int64_t nnz_cap);

/* The whole hot path in one call: selection (as vecattn_select) followed by
 * vector-sparse attention (as vecattn_sparse_fwd) over that selection, without the
 * CSR round trip -- the attention plan (per 256-row item: the union of its blocks'
 * selections with per-block membership) is built directly from the on-chip-produced
 * selection bitmask.  `offsets` and `*d_nnz` are always written; `indices` (CSR, may
 * be NULL with cap = 0) is written iff nnz <= cap.  The attention runs iff
 * nnz <= nnz_cap (the workspace's plan capacity); otherwise o/lse are untouched and the
 * caller reads d_nnz, grows the workspace and calls again.
 * Streams: for non-causal problems the CSR emission runs on a library-owned side stream
 * beside the attention kernel.  It is forked from `stream` with an event after the plan
 * and joined back into `stream` with an event before the call's work ends. Every output is
 * therefore complete when `stream` reaches that point.  The side stream is one per device,
 * shared by all callers (host calls serialise on it).  While `stream` is being captured into
 * a CUDA graph the emission stays on `stream`, so a capture never includes the shared side
 * stream.  Setting VECATTN_SERIAL_EMIT=1 emits on `stream` always.                */
VECATTN_API vecattn_status_t vecattn_forward(const vecattn_problem_t* p, const vecattn_select_params_t* s,
                                             const void* q, const void* k, const void* v, int64_t* offsets,
                                             int32_t* indices, int64_t cap, int64_t* d_nnz, int64_t nnz_cap,
                                             void* o, float* lse, void* ws, size_t ws_bytes,
                                             vecattn_stream_t stream);

/* ------------------------------------------- fused attention + all-gather */

/* Output replication: the head-parallel output all-gather of the multi-GPU path (SURVEY
 * 8(e) C1b) fused into the attention epilogue.  Every O row this call
 * produces is stored straight into the full-size O buffer of every rank -- by P2P stores
 * over NVLink into each peer's buffer (peer_o), or by one NVLS multicast store
 * (multimem.st) when o_multicast is set -- instead of being all-gathered after the kernel.
 * Row (b, h, r) of the call (h < p->Hq, the call's local query heads) lands at row
 * ((b * heads_total + head0 + h) * N + r) of each [B, heads_total, N, D] bf16 buffer.
 * The buffers are device addresses valid in the calling process (e.g. the peer mappings of a
 * torch symmetric-memory allocation); they are written, never read.  The stores are weak:
 * the caller orders them before any rank reads O (a cross-rank barrier after the call).
 * Ownership stays with the caller; the library keeps no reference after the call.   */
typedef struct {
    int32_t n_peers;     /* 0..8 entries of peer_o (the caller's own buffer included)          */
    void* peer_o[8];     /* 16-byte aligned device addresses of each rank's full O             */
    void* o_multicast;   /* NVLS multicast address of the full O or NULL (then peer_o is used) */
    int64_t head0;       /* first global query head of this call's heads, >= 0                 */
    int64_t heads_total; /* query heads of the full O, >= head0 + p->Hq                         */
    int64_t item_begin;  /* work window over the call's 256-row attention items, flattened as  */
    int64_t item_end;    /* (b*Hq + h) * ceil(N/256) + r/256: only rows of items in            */
                         /* [item_begin, item_end) are computed and stored (O, replicas, LSE); */
                         /* item_end <= 0 = every item.  The selection (offsets/indices) still */
                         /* covers every row of the call.                                       */
} vecattn_replica_t;

/* vecattn_forward with output replication.  `o` may be NULL (no local compact copy); if
 * non-NULL it is written as by vecattn_forward.  rep == NULL or (n_peers == 0 and
 * o_multicast == NULL) behaves exactly as vecattn_forward.  Errors: INVALID_ARGUMENT for
 * n_peers outside 0..8, a NULL peer, head0 < 0 or head0 + p->Hq > heads_total, a work
 * window outside [0, B*Hq*ceil(N/256)] or empty, or o == NULL without a replica; SHAPE for a
 * peer/multicast address not 16-byte aligned.  The work window is the flattened (head, block)
 * partition of SURVEY 8(e): ranks split B*H*ceil(N/256) items evenly, each calling with the
 * heads its window touches.  The CTA-pair kernel (VECATTN_PAIR=1) is not used with replicas
 * or windows.                                                                           */
VECATTN_API vecattn_status_t vecattn_forward_replicated(const vecattn_problem_t* p, const vecattn_select_params_t* s,
                                                        const void* q, const void* k, const void* v,
                                                        int64_t* offsets, int32_t* indices, int64_t cap,
                                                        int64_t* d_nnz, int64_t nnz_cap, void* o, float* lse,
                                                        const vecattn_replica_t* rep, void* ws, size_t ws_bytes,
                                                        vecattn_stream_t stream);

/* ------------------------------------------------------------- reference */

VECATTN_API size_t vecattn_dense_workspace_bytes(const vecattn_problem_t* p);

/* Dense attention, Eq. 1, same kernel skeleton with contiguous K/V tiles
 * (the speed-up denominator).  lse may be NULL.                                     */
VECATTN_API vecattn_status_t vecattn_dense_fwd(const vecattn_problem_t* p, const void* q, const void* k, const void* v,
                                   void* o, float* lse, void* ws, size_t ws_bytes, vecattn_stream_t stream);

/* ------------------------------------------------ per-head filter ratios (Eq. 4) */

/* Dynamic programming for the offline search of per-head filter ratios, Eq. 4.
 * Host-only: no GPU work, callable without a device.  sp and perf are row-major HOST arrays
 * [H][n_cand]: the sparsity sp_h(alpha_c) in [0, 1] and the performance Perf_h(alpha_c) of
 * head h under candidate filter ratio c, recorded offline by sampling.
 * DP[h][rho] of Eq. 4 -- the best total performance of the first h heads at average
 * sparsity rho -- is run on the running sparsity sum h*rho, quantised to 1/grid (round half
 * up), with the target read as a floor: the result maximises sum_h Perf_h(alpha_h) subject
 * to (1/H) sum_h sp_h(alpha_h) >= rho_target (reading R17b).  Among optimal
 * assignments the lexicographically smallest candidate sequence is returned.
 * Writes choice[H] (candidate index per head) and *best (the optimal total performance).
 * Errors: VECATTN_ERR_INVALID_ARGUMENT for NULL pointers, H < 1, n_cand < 1, grid < 1,
 * rho_target outside [0, 1], non-finite or out-of-range inputs, or when no assignment
 * reaches the target (then *best = -inf and choice is untouched).  O(H * n_cand * H * grid). */
VECATTN_API vecattn_status_t vecattn_alpha_dp(int32_t H, int32_t n_cand, const float* sp, const float* perf,
                                              float rho_target, int32_t grid, int32_t* choice, double* best);

/* ------------------------------------------------ naive selection baselines */

/* The paper's NAIVE materialise-then-filter selection (Fig. 5), the
 * comparison baseline for the fused vecattn_select.  The pooled
 * score map S_p = Q_p K^T (fp32, [B*Hq*N_p, N]) is written to the workspace in HBM and
 * filtered row by row:
 *   VECATTN_NAIVE_MINS  Eq. 3 with the global row max: the same index sets as
 *                       vecattn_select(VECATTN_SEL_MINS_EXACT) with the same alpha.
 *   VECATTN_NAIVE_TOPP  topP: per row softmax(scale * s) over the
 *                       visible keys, keys sorted by descending probability (ties -> lowest
 *                       index), the smallest prefix whose cumulative mass is >= top_p; keys
 *                       of zero (fp32) probability are never taken.
 * Arguments, CSR layout, capacity protocol and causal rule as vecattn_select (indices may be
 * NULL with cap = 0 for counts only).  alpha >= 0 (MINS), 0 < top_p <= 1 (TOPP); pq in {64,
 * 128}.  The workspace (vecattn_select_naive_workspace_bytes) holds the 4*R*N-byte score map
 * and, for TOPP, sort buffers for up to 2^29 keys at a time; errors as vecattn_select.      */
typedef enum { VECATTN_NAIVE_MINS = 0, VECATTN_NAIVE_TOPP = 1 } vecattn_naive_mode_t;
VECATTN_API size_t vecattn_select_naive_workspace_bytes(const vecattn_problem_t* p, int32_t pq, int32_t mode);
VECATTN_API vecattn_status_t vecattn_select_naive(const vecattn_problem_t* p, int32_t pq, int32_t mode, float alpha,
                                                  float top_p, const void* q, const void* k, int64_t* offsets,
                                                  int32_t* indices, int64_t cap, int64_t* d_nnz, void* ws,
                                                  size_t ws_bytes, vecattn_stream_t stream);

/* ----------------------------------------------------------- diagnostics */

/* Test hook: writes d_bad[0] = number of CSR rows violating ascending/unique/range/
 * causal rules (device int32).                                                      */
VECATTN_API vecattn_status_t vecattn_validate_selection(const vecattn_problem_t* p, int32_t pq, const int64_t* offsets,
                                            const int32_t* indices, int32_t* d_bad, vecattn_stream_t stream);

/* Test hook: the raw pooled-score accumulators <Q_p[i], k_j> (fp32, unscaled) of the
 * selection GEMM, scores [B*Hq*N_p, N]; ws sized by vecattn_select_workspace_bytes
 * with the same pq.                                                                  */
VECATTN_API vecattn_status_t vecattn_debug_scores(const vecattn_problem_t* p, int32_t pq, const void* q, const void* k,
                                      float* scores, void* ws, size_t ws_bytes, vecattn_stream_t stream);

/* Measurement hook (bench.py roofline).  When enabled, every vecattn_forward /
 * vecattn_sparse_fwd / vecattn_dense_fwd call records CUDA events on its stream around
 * (a) query pooling + the selection GEMM/filter + offsets scan, (b) CSR emission + the
 * attention plan, and (c) the attention kernel alone.  Library-owned events, one set per
 * process (not thread-safe; for benchmarking only).  vecattn_kernel_timing_last waits for
 * the events of the most recent timed call and returns the three durations in ms (-1 for a
 * stage the call did not run).  Disabled by default: no events are recorded.            */
VECATTN_API vecattn_status_t vecattn_kernel_timing(int32_t enable);
VECATTN_API vecattn_status_t vecattn_kernel_timing_last(float* select_ms, float* plan_ms, float* attn_ms);

VECATTN_API const char* vecattn_status_string(vecattn_status_t s);
/* Text of the last CUDA error that made an entry point return VECATTN_ERR_CUDA (this thread). */
VECATTN_API const char* vecattn_last_cuda_error(void);
VECATTN_API int32_t vecattn_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* VECATTN_H */
