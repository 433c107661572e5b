// common.cuh — sm_100a device primitives for the VecAttention hot path.
//
// Thin inline-PTX wrappers: mbarrier, TMA (tile + tile::gather4), tcgen05
// (alloc / mma kind::f16 / commit / ld / st / fences) and UMMA shared-memory and
// instruction descriptors.  Bit layouts follow the PTX ISA 8.6+ tcgen05 chapter
// (descriptor fields cross-checked against CuTe's UMMA::SmemDescriptor /
// UMMA::InstrDescriptor in cute/arch/mma_sm100_desc.hpp).  No oracle code here.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#define VA_DEV __device__ __forceinline__

namespace va {

// ----------------------------------------------------------------------------- misc
VA_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

VA_DEV uint32_t warp_id() { return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0); }
VA_DEV uint32_t lane_id() { return threadIdx.x & 31u; }

VA_DEV bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(pred));
    return pred != 0;
}

// ------------------------------------------------------------------------- mbarrier
VA_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
VA_DEV void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// Named barrier `id` (1..15) over `n` threads (a multiple of 32) of the CTA.
VA_DEV void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
VA_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

VA_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
VA_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// Predicated forms for warp-wide code: only lanes with pred != 0 arrive, and the warp does not
// branch (a single-lane `if` around an arrive costs a divergent branch and reconvergence in
// the hot loops).
VA_DEV void mbar_arrive_if(uint64_t* bar, uint32_t pred) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n"
        " @p mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n}" ::"r"(smem_u32(bar)),
        "r"(pred)
        : "memory");
}
VA_DEV void mbar_arrive_expect_tx_if(uint64_t* bar, uint32_t bytes, uint32_t pred) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n"
        " @p mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n}" ::"r"(smem_u32(bar)),
        "r"(bytes), "r"(pred)
        : "memory");
}
VA_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// VA_WAIT_HINT_NS (build knob): suspend-time hint of the try_wait in mbar_wait (0 = the
// system default).  Without a hint a waiting thread re-polls every few ns, and a warp that waits
// for long (a scheduler waiting out an item, a softmax waiting for S) spends issue slots its SMSP
// neighbours need; with one the thread sleeps until the phase completes or the hint expires.
#ifndef VA_WAIT_HINT_NS
#define VA_WAIT_HINT_NS 100000
#endif
VA_DEV bool mbar_try_wait_hint(uint64_t* bar, uint32_t parity, uint32_t hint_ns) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(hint_ns)
        : "memory");
    return ok != 0;
}
VA_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    if constexpr (VA_WAIT_HINT_NS > 0) {
        while (!mbar_try_wait_hint(bar, parity, VA_WAIT_HINT_NS)) {
        }
    } else {
        while (!mbar_try_wait(bar, parity)) {
        }
    }
}
// Long waits (a warp idling for most of an item): always with a suspend-time hint.
VA_DEV void mbar_wait_long(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait_hint(bar, parity, 1000000u)) {
    }
}

// ------------------------------------------------------------------------------ TMA
VA_DEV void tma_prefetch_desc(const void* desc) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(desc) : "memory");
}
// 3-D tile load: coordinates {c0 (innermost, elements), c1, c2}.
VA_DEV void tma_load_3d(void* dst, const void* desc, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// 3-D tile load with an L2 cache-policy hint (createpolicy value).
VA_DEV void tma_load_3d_hint(void* dst, const void* desc, uint64_t* bar, int c0, int c1, int c2, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}
VA_DEV uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// 2-D row gather: 4 rows (r0..r3) x box-width columns starting at column c0.
VA_DEV void tma_gather4(void* dst, const void* desc, uint64_t* bar, int c0, int r0, int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

// -------------------------------------------------------------------------- tcgen05
template <uint32_t NCOLS>
VA_DEV void tmem_alloc(uint32_t* smem_dst) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "n"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <uint32_t NCOLS>
VA_DEV void tmem_dealloc(uint32_t taddr) {  // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS));
}
VA_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
VA_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem desc] * B[smem desc]
VA_DEV void mma_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]
VA_DEV void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on an mbarrier when all previously issued tcgen05.mma of this thread complete.
VA_DEV void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// 32 lanes x 32-bit, 32 consecutive columns per thread.
VA_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
// 32 lanes x 32-bit, 8 consecutive columns per thread.
VA_DEV void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
VA_DEV void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
VA_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
VA_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

VA_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
// 32 lanes x 32 consecutive columns of zeros.
VA_DEV void tmem_st32_zero(uint32_t taddr) {
    const uint32_t z = 0u;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(z)
        : "memory");
}
VA_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ UMMA descriptors
// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"):
//   [0,14)  start address >> 4      [16,30) leading byte offset >> 4
//   [32,46) stride byte offset >> 4 [46,48) version = 1 (sm_100)
//   [49,52) base offset = 0          [52]    lbo mode = 0
//   [61,64) layout: 2 = SWIZZLE_128B
// K-major SW128 (rows of 128 B, 8-row atoms of 1024 B): LBO unused (=16 B), SBO = 1024 B.
// MN-major SW128 (128 B = 64 elements along MN, rows along K): LBO = byte stride between
// 64-element MN blocks, SBO = byte stride between 8-row K groups (1024 B here).
VA_DEV uint64_t make_sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout = 2u) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1u << 46;       // version
    d |= (uint64_t)layout << 61;   // 2 = SWIZZLE_128B, 0 = SWIZZLE_NONE (interleaved core matrices)
    return d;
}
// K-major SWIZZLE_NONE layout of a [rows x 16] bf16 tile: 8x8 core matrices (128 B each),
// element (r, e) at ((r/8)*2 + e/8)*128 + (r%8)*16 + (e%8)*2; K-direction core stride (LBO)
// 128 B, 8-row-group stride (SBO) 256 B.
VA_DEV uint32_t k16_offset(int r, int e) { return ((r >> 3) * 2 + (e >> 3)) * 128 + (r & 7) * 16 + (e & 7) * 2; }
// Instruction descriptor, kind::f16 with bf16 A/B and f32 accumulate:
//   [4,6) c_format=1 (F32)  [7,10) a_format=1 (BF16)  [10,13) b_format=1 (BF16)
//   [15] a_major (0=K,1=MN) [16] b_major  [17,23) N>>3  [24,29) M>>4
constexpr uint32_t make_idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ------------------------------------------------------- CTA pair (cta_group::2, cluster of 2)
// Semantics checked on the B200 by scripts/probe_pair.cu: for an M = 256 pair MMA, CTA r
// holds A rows [128r, 128r+128) (its own smem / TMEM) and B rows (N index) [N/2 r, N/2 (r+1));
// each CTA's TMEM receives its 128 rows x all N columns.  A gather4 with .cta_group::2 may
// complete on the peer CTA's mbarrier.
VA_DEV uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
VA_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> shared::cluster address of the same offset in CTA `rank`
VA_DEV uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
VA_DEV void mbar_arrive_cluster(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
// Remote arrive without release semantics (scripts/probe_sync.cu: ~95 ns one way vs ~240 ns
// for .release.cluster in isolation, far more under load).  Only for hand-offs whose data is
// already complete from the issuing thread's view (tcgen05.wait::st / ::ld, a register value).
VA_DEV void mbar_arrive_cluster_relaxed(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
VA_DEV bool mbar_try_wait_cl(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Non-blocking probe (test_wait never suspends the thread, unlike try_wait): for polling
// several barriers from one thread.  CTA-scope acquire: after a successful probe of a
// barrier completed from the peer CTA, follow with fence_acq_rel_cluster().
VA_DEV bool mbar_test_cl(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
VA_DEV bool mbar_test_cl(uint64_t* bar, uint32_t parity);
// Cluster-scope wait.  The phase of a pair barrier is often completed from the other SM
// (remote arrive, multicast commit); a suspended try_wait is not woken promptly by those
// (scripts/trace_pair.py: ~2 us late), so this spins on the non-suspending test_wait.
VA_DEV void fence_acq_rel_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
VA_DEV void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait_cl(bar, parity)) {
    }
}
VA_DEV void st_cluster_u32(uint32_t addr_cluster, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr_cluster), "r"(v) : "memory");
}
// 2-D row gather into this CTA's smem, completing on the mbarrier at `bar_cluster` (either CTA of the pair)
VA_DEV void tma_gather4_pair(void* dst, const void* desc, uint32_t bar_cluster, int c0, int r0, int r1, int r2,
                             int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.cta_group::2"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(desc), "r"(bar_cluster), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}
VA_DEV void tma_load_3d_pair_hint(void* dst, const void* desc, uint32_t bar_cluster, int c0, int c1, int c2,
                                  uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(desc), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}
template <uint32_t NCOLS>
VA_DEV void tmem_alloc_pair(uint32_t* smem_dst) {  // one warp in EACH CTA of the pair
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "n"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <uint32_t NCOLS>
VA_DEV void tmem_dealloc_pair(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS));
}
// Pair MMA (issued by the leader CTA only): D[tmem, both CTAs] (+)= A[smem] B[smem]
VA_DEV void mma2_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Pair MMA with A from each CTA's TMEM
VA_DEV void mma2_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive (once) on the mbarrier at the same offset in both CTAs when the issuing thread's MMAs complete.
VA_DEV void mma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

// ----------------------------------------------------------------------- numerics
VA_DEV float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
VA_DEV uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
// Packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2 process two fp32 lanes per instruction).
VA_DEV uint64_t pack_f32x2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
VA_DEV float2 unpack_f32x2(uint64_t v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
VA_DEV uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
VA_DEV float2 fadd2(float2 a, float2 b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pack_f32x2(a.x, a.y)), "l"(pack_f32x2(b.x, b.y)));
    return unpack_f32x2(d);
}
// exp2 on the FMA pipe for two lanes (FA4-style MUFU offload): round-to-nearest split
// x = i + f (f in [-0.5, 0.5]) via the 1.5*2^23 magic add, 2^f by a degree-3 minimax
// polynomial (max relative error 1.0e-4, well below bf16's 2^-9), 2^i by an integer add
// to the exponent field.  Inputs below -125 give exactly 0.
VA_DEV float2 ex2_poly2(float x0_in, float x1_in) {
    const float x0 = fmaxf(x0_in, -125.f);
    const float x1 = fmaxf(x1_in, -125.f);
    const uint64_t X = pack_f32x2(x0, x1);
    const uint64_t T = ffma2(X, pack_f32x2(1.f, 1.f), pack_f32x2(12582912.f, 12582912.f));
    const uint64_t R = ffma2(T, pack_f32x2(1.f, 1.f), pack_f32x2(-12582912.f, -12582912.f));
    const uint64_t F = ffma2(R, pack_f32x2(-1.f, -1.f), X);
    uint64_t P = ffma2(F, pack_f32x2(0.054993368685245514f, 0.054993368685245514f),
                       pack_f32x2(0.24221104383468628f, 0.24221104383468628f));
    P = ffma2(P, F, pack_f32x2(0.693286120891571f, 0.693286120891571f));
    P = ffma2(P, F, pack_f32x2(1.f, 1.f));
    const float2 p = unpack_f32x2(P), t = unpack_f32x2(T);
    // exact 0 below the clamp (masked scores are -inf / -2^100; like ex2.approx.ftz, which flushes)
    return make_float2(x0_in < -125.f ? 0.f : __uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                       x1_in < -125.f ? 0.f : __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}
// Leaner FMA-pipe exp2 for two lanes (10 instructions per pair instead of 12): the same
// split and polynomial as ex2_poly2, inputs clamped at -125 and NOT flushed to zero below it,
// so a masked score (-inf, -2^100 scale) gives 2^-125 ~ 2.4e-38 instead of 0 -- a contribution
// ~1e-38 of a row's mass (l >= 1 after the max shift), far below bf16/fp32 resolution.
VA_DEV float2 ex2_poly2_fast(float x0_in, float x1_in) {
    const uint64_t X = pack_f32x2(fmaxf(x0_in, -125.f), fmaxf(x1_in, -125.f));
    const uint64_t T = ffma2(X, pack_f32x2(1.f, 1.f), pack_f32x2(12582912.f, 12582912.f));
    const uint64_t R = ffma2(T, pack_f32x2(1.f, 1.f), pack_f32x2(-12582912.f, -12582912.f));
    const uint64_t F = ffma2(R, pack_f32x2(-1.f, -1.f), X);
    uint64_t P = ffma2(F, pack_f32x2(0.054993368685245514f, 0.054993368685245514f),
                       pack_f32x2(0.24221104383468628f, 0.24221104383468628f));
    P = ffma2(P, F, pack_f32x2(0.693286120891571f, 0.693286120891571f));
    P = ffma2(P, F, pack_f32x2(1.f, 1.f));
    const float2 p = unpack_f32x2(P), t = unpack_f32x2(T);
    return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                       __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}
// Order-preserving map fp32 -> u32 (a < b  <=>  key(a) < key(b) for non-NaN).
VA_DEV uint32_t f32_order_key(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
VA_DEV float f32_from_order_key(uint32_t k) {
    uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
    return __uint_as_float(u);
}

}  // namespace va
