// Cross-SM signalling latency inside a CTA pair (cluster of 2), for the pair attention kernel:
//   A: remote mbarrier arrive ping-pong (leader <-> peer), per wait flavour
//   B: tcgen05.commit multicast after one pair MMA: when does each CTA observe its barrier?
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o probe_sync probe_sync.cu
#include "../paper_2603_29494_b200/csrc/common.cuh"
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

using namespace va;

VA_DEV long long gt() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
VA_DEV bool test_acq_cluster(uint64_t* bar, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(smem_u32(bar)), "r"(par) : "memory");
    return ok;
}
VA_DEV bool test_relaxed(uint64_t* bar, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(smem_u32(bar)), "r"(par) : "memory");
    return ok;
}
VA_DEV bool try_acq_cluster(uint64_t* bar, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(smem_u32(bar)), "r"(par) : "memory");
    return ok;
}
VA_DEV bool try_acq_cta(uint64_t* bar, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(smem_u32(bar)), "r"(par) : "memory");
    return ok;
}
template <int W>
VA_DEV void waitf(uint64_t* bar, uint32_t par) {
    if (W == 0) while (!try_acq_cluster(bar, par)) {}
    if (W == 1) while (!test_acq_cluster(bar, par)) {}
    if (W == 2) { while (!test_relaxed(bar, par)) {} asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
    if (W == 3) while (!try_acq_cta(bar, par)) {}
    if (W == 4) while (!test_relaxed(bar, par)) {}
}
VA_DEV void arrive_relaxed_cluster(uint32_t a) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}

template <int W, int REL>
__global__ void __cluster_dims__(2, 1, 1) pingpong(long long* out, int iters) {
    __shared__ uint64_t bar;
    const uint32_t rank = cluster_rank();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    cluster_sync_all();
    const uint32_t other = mapa_rank(smem_u32(&bar), rank ^ 1u);
    if (threadIdx.x == 0) {
        long long t0 = gt();
        for (int i = 0; i < iters; ++i) {
            if (rank == 0) {
                if (REL) arrive_relaxed_cluster(other); else mbar_arrive_cluster(other);
                waitf<W>(&bar, i & 1);
            } else {
                waitf<W>(&bar, i & 1);
                if (REL) arrive_relaxed_cluster(other); else mbar_arrive_cluster(other);
            }
        }
        if (rank == 0) out[0] = gt() - t0;
    }
    cluster_sync_all();
}

// B: 64 rounds of { leader: one pair MMA M256 N64 K16 + multicast commit; both CTAs: observe } with
// the leader's observing thread polling with flavour W; record observation times in both CTAs.
template <int W>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) commit_lat(long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
    uint64_t* go = bar + 1;
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 32768 + 64);
    const uint32_t rank = cluster_rank();
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 8192; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(go, 1); fence_barrier_init(); }
    fence_proxy_async();
    if (warp == 0) tmem_alloc_pair<512>(slot);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tm = *slot;
    const uint32_t idesc = make_idesc_bf16(256, 64, 0, 0);
    const uint64_t ad = make_sdesc(smem_u32(smem), 16, 1024), bd = make_sdesc(smem_u32(smem + 16384), 16, 1024);
    for (int i = 0; i < 64; ++i) {
        if (rank == 0 && warp == 1 && elect_one()) {
            const long long t0 = gt();
            mma2_bf16_ss(tm, ad, bd, idesc, 0);
            mma_commit_pair(bar);
            waitf<W>(bar, i & 1);
            out[3 * i + 0] = t0;
            out[3 * i + 1] = gt();
        }
        if (rank == 1 && warp == 2 && threadIdx.x == 64) {
            waitf<1>(bar, i & 1);
            out[3 * i + 2] = gt();
        }
        tc_fence_before();
        cluster_sync_all();
        tc_fence_after();
    }
    cluster_sync_all();
    if (warp == 0) tmem_dealloc_pair<512>(tm);
}

template <typename K>
static void run_pp(K k, const char* name, long long* d) {
    const int iters = 2000;
    k<<<2, 32>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long ns;
    cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
    printf("ping-pong %-40s %s round trip %.0f ns\n", name, cudaGetErrorString(e), (double)ns / iters);
}
template <int W>
static void run_commit(const char* name, long long* d) {
    cudaFuncSetAttribute(commit_lat<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    commit_lat<W><<<2, 128, 40000>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(192);
    cudaMemcpy(h.data(), d, 192 * 8, cudaMemcpyDeviceToHost);
    std::vector<long long> lead, peer;
    for (int i = 4; i < 64; ++i) {
        lead.push_back(h[3 * i + 1] - h[3 * i]);
        peer.push_back(h[3 * i + 2] - h[3 * i]);
    }
    std::sort(lead.begin(), lead.end());
    std::sort(peer.begin(), peer.end());
    printf("commit   %-40s %s issue->leader sees %lld ns, issue->peer sees %lld ns (medians)\n", name,
           cudaGetErrorString(e), lead[lead.size() / 2], peer[peer.size() / 2]);
}

int main() {
    long long* d;
    cudaMalloc(&d, 4096);
    run_pp(pingpong<0, 0>, "try_wait.acquire.cluster / arrive.release", d);
    run_pp(pingpong<1, 0>, "test_wait.acquire.cluster / arrive.release", d);
    run_pp(pingpong<2, 0>, "test_wait.relaxed + fence / arrive.release", d);
    run_pp(pingpong<3, 0>, "try_wait.acquire.cta / arrive.release", d);
    run_pp(pingpong<4, 1>, "test_wait.relaxed / arrive.relaxed", d);
    run_pp(pingpong<1, 1>, "test_wait.acquire.cluster / arrive.relaxed", d);
    run_commit<0>("leader try_wait.acquire.cluster", d);
    run_commit<1>("leader test_wait.acquire.cluster", d);
    run_commit<2>("leader test_wait.relaxed + fence", d);
    run_commit<3>("leader try_wait.acquire.cta", d);
    return 0;
}
