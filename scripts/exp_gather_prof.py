import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_29494_b200.vecattn as va
N, H, D, pq = 32768, 8, 128, 64
q = torch.randn(1, H, N, D, device="cuda").bfloat16(); k = torch.randn_like(q); v = torch.randn_like(q)
Np = N // pq
sel = torch.arange(0, N, 2, device="cuda")
idx = sel.int().repeat(H * Np); off = torch.arange(0, H * Np + 1, device="cuda", dtype=torch.int64) * sel.numel()
for _ in range(2): va.sparse_fwd(q, k, v, off, idx, pq=pq)
torch.cuda.synchronize()
