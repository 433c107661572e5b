"""Experiment: sparse-attention throughput vs per-head K/V working set (L2 capacity)."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_29494_b200.vecattn as va

def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

H, D, pq = 4, 128, 64
for N in [32768, 65536, 131072, 262144]:
    q = torch.randn(1, H, N, D, device="cuda").bfloat16()
    k = torch.randn(1, H, N, D, device="cuda").bfloat16()
    v = torch.randn(1, H, N, D, device="cuda").bfloat16()
    Np = N // pq
    g = torch.Generator(device="cuda"); g.manual_seed(0)
    for frac, span in [(0.125, 1.0), (0.125, 0.5), (0.125, 0.25)]:
        nsel = int(N * frac)
        sel = torch.sort(torch.randperm(int(N * span), device="cuda", generator=g)[:nsel]).values
        idx = sel.int().repeat(H * Np)
        off = torch.arange(0, H * Np + 1, device="cuda", dtype=torch.int64) * nsel
        ws = va.Workspace("cuda")
        t = timeit(lambda: va.sparse_fwd(q, k, v, off, idx, pq=pq, ws=ws))
        f = 4.0 * N * nsel * D * H
        print(f"N={N:7d} sel={frac} span={span} (K/V working set {int(N*span)*D*4/1e6:.0f} MB/head): "
              f"{t:.2f} ms {f/t/1e9:.0f} TFLOP/s", flush=True)
    del q, k, v, idx
