"""Experiment: sparse throughput vs K/V working set with DISTINCT random lists per block."""
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

H, D, pq, N = 4, 128, 64, 131072
q = torch.randn(1, H, N, D, device="cuda").bfloat16()
k = torch.randn(1, H, N, D, device="cuda").bfloat16()
v = torch.randn(1, H, N, D, device="cuda").bfloat16()
Np = N // pq
nsel = 8192
g = torch.Generator(device="cuda"); g.manual_seed(0)
for span in [16384, 32768, 65536, 131072]:
    # each block: nsel distinct keys from [0, span) -- random, different per block;
    # adjacent blocks (same 256-row item) share half their keys
    r = torch.rand(H * Np // 2, span, device="cuda", generator=g)
    base = torch.topk(r, nsel, dim=1).indices
    sels = []
    for b in range(H * Np):
        s_ = base[b // 2]
        sels.append(torch.sort(s_).values)
    idx = torch.cat(sels).int()
    off = torch.arange(0, H * Np + 1, device="cuda", dtype=torch.int64) * nsel
    ws = va.Workspace("cuda")
    t = timeit(lambda: va.sparse_fwd(q, k, v, off, idx, pq=pq, ws=ws))
    f = 4.0 * N * nsel * D * H
    print(f"span={span:7d} (K/V working set/head {span*D*4/1e6:.0f} MB): {t:.2f} ms {f/t/1e9:.0f} TFLOP/s", flush=True)
