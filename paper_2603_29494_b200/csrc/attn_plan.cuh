// attn_plan.cuh — walking an attention item's key plan, shared by the two attention
// kernels (attn.cu, attn_db.cu).  Internal to the library; no oracle code.
//
// A work item is 256 query rows (two M=128 tiles) of one head.  Its plan (built by
// plan_kernel / worklist_kernel) is the union of the item's block index lists in three
// sorted segments -- keys of both tiles, tile 0 only, tile 1 only -- cut into chunks of
// CHUNK keys; the dense path walks contiguous key chunks instead.
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace va {
namespace plan {

// Debug timeline (p.trace != null, [32][4096] int64): CTAs 0 and 1 record %globaltimer (ns) per chunk and event kind
// (0 K issue, 1 V issue, 2 K landed, 3 V landed, 4/5 PV0/PV1 issued, 6/7 S0 ready/P0 done,
// 8/9 S1 ready/P1 done) -- scripts/trace_run.py.
constexpr int kTraceChunks = 4096;
// %globaltimer (ns), comparable across the SMs of a pair (clock64 is per SM)
VA_DEV long long globaltimer_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Compiled in only with -DVA_TRACE=1 (scripts/trace_*.py builds: scripts/build_variant.py
// <tag> <file> -DVA_TRACE=1); the production kernels carry no timeline code.
#ifndef VA_TRACE
#define VA_TRACE 0
#endif
VA_DEV void trace(const AttnParams& p, int kind, int64_t c) {
    if constexpr (VA_TRACE != 0) {
        if (p.trace != nullptr && blockIdx.x < 2 && c < kTraceChunks)  // CTA 1 (the pair's peer): kinds + 16
            p.trace[(int64_t)(kind + 16 * blockIdx.x) * kTraceChunks + c] = globaltimer_ns();
    }
}

// Dynamic item scheduler.  die_mode 0: one atomic counter over the head-major item order.
// die_mode 1/2: one counter per die of the GPU (two L2 halves); die d walks the heads
// h = d, d+2, ... so each die's L2 holds the K/V of fewer heads, and takes the other die's
// items once its own are gone.  Returns an item index >= total_items when all are done.
VA_DEV int next_item(const AttnParams& p) {
    if (p.die_mode == 0) return atomicAdd(p.work_counter, 1);
    uint32_t smid, nsm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(nsm));
    const int d0 = p.die_mode == 1 ? (smid >= nsm / 2 ? 1 : 0) : (int)(smid & 1u);
    for (int t = 0; t < 2; ++t) {
        const int d = d0 ^ t;
        const int li = atomicAdd(p.work_counter + d, 1);
        const int64_t head = 2 * (li / p.n_mt) + d;
        if (head < p.BH) return (int)(head * p.n_mt + li % p.n_mt);
    }
    return (int)p.total_items;
}

struct Item {
    int64_t bh, it;  // head, 256-row item within the head
    int n_chunks;
    int lb, l0, l1;  // gather: plan segment lengths (keys of both tiles | tile 0 only | tile 1 only)
    int nb, n0, n1;  // gather: chunks per segment
    int len;         // dense: key extent
    int64_t base;    // gather: plan base
};

struct Chunk {
    int mask;   // bit t: tile t computes this chunk
    int start;  // first plan entry (relative to the item base) / first key (dense)
    int len;    // valid entries / keys
};

template <int kChunk, bool GATHER>
VA_DEV Item decode_item(const AttnParams& p, int item) {
    Item I;
    // scheduler position -> item (bh * n_mt + it).  Longest-first within a head: causal items
    // by position (reversed); with p.item_order (written after the plan), non-causal plans by
    // their tile-chunk counts, and work windows (vecattn_replica_t) over the window's items.
    const int64_t x = p.item_order != nullptr ? (int64_t)p.item_order[item]
                                              : (item / p.n_mt) * p.n_mt + (p.n_mt - 1 - (item % p.n_mt));
    I.bh = x / p.n_mt;
    I.it = x % p.n_mt;
    if constexpr (GATHER) {
        const int64_t G = 256 / p.pq;
        const int64_t x = I.bh * p.n_mt + I.it;
        I.lb = p.wl_len[3 * x];
        I.l0 = p.wl_len[3 * x + 1];
        I.l1 = p.wl_len[3 * x + 2];
        I.nb = (I.lb + kChunk - 1) / kChunk;
        I.n0 = (I.l0 + kChunk - 1) / kChunk;
        I.n1 = (I.l1 + kChunk - 1) / kChunk;
        I.n_chunks = I.nb + I.n0 + I.n1;
        I.base = p.offsets[I.bh * p.Np + G * I.it];
        I.len = 0;
    } else {
        const int64_t kend = p.causal ? min(p.N, (I.it + 1) * 256) : p.N;
        I.len = (int)kend;
        I.base = 0;
        I.n_chunks = (int)((kend + kChunk - 1) / kChunk);
        I.lb = I.l0 = I.l1 = I.nb = I.n0 = I.n1 = 0;
    }
    return I;
}

// Chunk order: shared chunks first, then tile-0-only and tile-1-only chunks interleaved
// (so the tensor core alternates between the two softmax warpgroups).
template <int kChunk, bool GATHER>
VA_DEV Chunk chunk_info(const Item& I, int j) {
    Chunk c;
    if constexpr (!GATHER) {
        c.mask = 3;
        c.start = kChunk * j;
        c.len = min(kChunk, I.len - kChunk * j);
        return c;
    } else {
        if (j < I.nb) {
            c.mask = 3;
            c.start = kChunk * j;
            c.len = min(kChunk, I.lb - kChunk * j);
            return c;
        }
        const int k = j - I.nb;
        const int m = min(I.n0, I.n1);
        int t, q;
        if (k < 2 * m) {
            t = k & 1;
            q = k >> 1;
        } else {
            t = I.n0 > I.n1 ? 0 : 1;
            q = m + (k - 2 * m);
        }
        c.mask = 1 << t;
        if (t == 0) {
            c.start = I.lb + kChunk * q;
            c.len = min(kChunk, I.l0 - kChunk * q);
        } else {
            c.start = I.lb + I.l0 + kChunk * q;
            c.len = min(kChunk, I.l1 - kChunk * q);
        }
        return c;
    }
}

// Position in the item of tile t's q-th chunk (gather plans): the shared chunks, then its own
// single-tile chunks -- interleaved with the other tile's, then the longer list's tail.
VA_DEV int own_chunk(const Item& I, int t, int q) {
    if (q < I.nb) return q;
    const int r = q - I.nb, m = min(I.n0, I.n1);
    return I.nb + (r < m ? 2 * r + t : 2 * m + (r - m));
}

// First chunk index > j that tile t computes (n_chunks if none).
template <bool GATHER>
VA_DEV int next_chunk(const Item& I, int t, int j) {
    if constexpr (!GATHER) {
        return j + 1;
    } else {
        const int n = I.n_chunks;
        const int mt = t == 0 ? I.n0 : I.n1;
        const int m = min(I.n0, I.n1);
        int x = j + 1;
        if (x < I.nb) return x;
        if (mt == 0) return n;
        // own chunks of tile t after the shared segment: interleaved k = 2q + t (q < m), then
        // (if t owns the longer list) the tail k >= 2m
        const int k = x - I.nb;
        if (k < 2 * m) {
            const int kk = ((k & 1) == t) ? k : k + 1;
            if (kk < 2 * m) return I.nb + kk;
            // past the interleave: the tail belongs to tile t only if its list is the longer
        }
        const bool tail_owner = (t == 0) ? (I.n0 > I.n1) : (I.n1 >= I.n0);
        if (!tail_owner || mt == m) return n;
        return max(x, I.nb + 2 * m);
    }
}

// ---------------------------------------------------------------- O output
// An O row goes to the call's own buffer (p.o, may be null) and, for the fused all-gather
// (vecattn_forward_replicated), to the same row of every rank's full O:
// P2P stores into each peer's buffer, or one multimem (NVLS multicast) store.
struct ORow {
    __nv_bfloat16* local;  // this row in p.o, or null
    int64_t grow;          // row index in the replica buffers
};
template <int D>
VA_DEV ORow o_row(const AttnParams& p, int64_t bh, int64_t qrow) {
    ORow r;
    r.local = p.o != nullptr ? p.o + (bh * p.N + qrow) * D : nullptr;
    const int64_t b = bh / p.Hq, h = bh % p.Hq;
    r.grow = (b * p.rep_heads + p.rep_head0 + h) * p.N + qrow;
    return r;
}
VA_DEV void multimem_st16(void* addr, uint4 w) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "r"(w.x), "r"(w.y),
                 "r"(w.z), "r"(w.w)
                 : "memory");
}
// 16 bytes (8 bf16) of row r at column col; streamed (evict-first) stores
template <int D>
VA_DEV void o_store16(const AttnParams& p, const ORow& r, int col, uint4 w) {
    if (r.local != nullptr) __stcs(reinterpret_cast<uint4*>(r.local + col), w);
    if (p.o_mc != nullptr) {
        multimem_st16(p.o_mc + r.grow * D + col, w);
    } else {
        for (int i = 0; i < p.rep_n; ++i) __stcs(reinterpret_cast<uint4*>(p.rep_o[i] + r.grow * D + col), w);
    }
}

}  // namespace plan
}  // namespace va
