"""Experiment: gather-path overhead. Sparse attention with synthetic CSR (all keys /
every 2nd key / random 25%) vs the dense kernel on the same shape."""
import sys, os, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_29494_b200.vecattn as va

def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

N, H, D, pq = int(sys.argv[1]) if len(sys.argv) > 1 else 32768, 8, 128, 64
q = torch.randn(1, H, N, D, device="cuda").bfloat16()
k = torch.randn(1, H, N, D, device="cuda").bfloat16()
v = torch.randn(1, H, N, D, device="cuda").bfloat16()
Np = N // pq
dense = timeit(lambda: va.dense_fwd(q, k, v))
fl = 4.0 * N * N * D * H
print(f"dense {dense:.2f} ms  {fl/dense/1e9:.0f} TFLOP/s")
g = torch.Generator(device="cuda"); g.manual_seed(0)
for name, sel in [("all", torch.arange(N, device="cuda")), ("stride2", torch.arange(0, N, 2, device="cuda")),
                  ("rand25", torch.sort(torch.randperm(N, device="cuda", generator=g)[: N // 4]).values)]:
    idx = sel.int().repeat(H * Np)
    off = torch.arange(0, H * Np + 1, device="cuda", dtype=torch.int64) * sel.numel()
    ws = va.Workspace("cuda")
    t = timeit(lambda: va.sparse_fwd(q, k, v, off, idx, pq=pq, ws=ws))
    f = 4.0 * N * sel.numel() * D * H
    print(f"sparse[{name}] {t:.2f} ms  {f/t/1e9:.0f} TFLOP/s  keys/blk={sel.numel()}")
