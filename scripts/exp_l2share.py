"""How much of the sparse attention time is L2 misses on K/V?  Same selection, same
compute: 24 query heads over ONE shared KV head (67 MB of K+V, L2-resident) vs over 24
identical copies of it (1.6 GB, the real footprint)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
dev = torch.device("cuda")
wl = synth.WORKLOADS["dit128k"]
N, D, H = wl.N, wl.D, int(sys.argv[1]) if len(sys.argv) > 1 else 24
dirs, kk, vv = synth.video_kv_head(N, D, wl.grid, synth.seed_of(wl.cfg_id, 0, 0, 1), dev)
q = torch.empty(1, H, N, D, dtype=torch.bfloat16, device=dev)
for h in range(H):
    g = torch.Generator(device=dev); g.manual_seed(synth.seed_of(wl.cfg_id, 0, h, 0))
    q[0, h] = (6.0 * dirs + torch.randn(N, D, generator=g, device=dev)).to(torch.bfloat16)
k1, v1 = kk.view(1, 1, N, D).contiguous(), vv.view(1, 1, N, D).contiguous()
kH, vH = k1.expand(1, H, N, D).contiguous(), v1.expand(1, H, N, D).contiguous()
cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=1.0039)
off, idx = va.select(q, kH, cfg)
torch.cuda.synchronize()
print("nnz", idx.numel(), "rho", 1 - idx.numel() * 64 / (H * N * N))
va.kernel_timing(True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for name, k, v in (("shared KV (Hkv=1)", k1, v1), ("24 copies (Hkv=H)", kH, vH)) * 2:
    ts = []
    for r in range(4):
        flush.zero_()
        o, lse = va.sparse_fwd(q, k, v, off, idx, pq=64)
        torch.cuda.synchronize()
        ts.append(va.kernel_timing_last()[2])
    print(f"{name}: attention ms {['%.2f' % t for t in ts]}")
