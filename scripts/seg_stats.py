"""Union-segment statistics of the sparse worklist on a bench workload (first H heads)."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
wl = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "dit128k"]
H = int(sys.argv[2]) if len(sys.argv) > 2 else 4
kind = sys.argv[3] if len(sys.argv) > 3 else "video"
alpha = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0039
dev = torch.device("cuda")
q, k, v = bench.build_inputs(wl, kind, dev, 0, H)
cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=alpha)
off, idx = va.select(q, k, cfg, causal=wl.causal)
pr = va.problem(q, k, wl.causal)
cap = idx.numel()
ws = torch.empty(va.sparse_workspace_bytes(pr, 64, cap), dtype=torch.uint8, device=dev)
o = torch.empty_like(q); lse = torch.empty(q.shape[:3], device=dev)
va.sparse_fwd_into(q, k, v, off, idx, 64, o, lse, ws, cap, wl.causal)
torch.cuda.synchronize()
base = (cap * 4 + 255) // 256 * 256
n_it = (wl.N + 255) // 256
lens = ws[base: base + H * n_it * 12].view(torch.int32).view(-1, 3).cpu().numpy().astype(np.int64)
lb, l0, l1 = lens[:, 0], lens[:, 1], lens[:, 2]
ch = lambda x: (x + 127) // 128
ch64 = lambda x: (x + 63) // 64
nnz = int(off[-1])
pairs = lb + l0, lb + l1
print(f"nnz={nnz} sum(lb)={lb.sum()} sum(l0)={l0.sum()} sum(l1)={l1.sum()}  both-fraction={lb.sum()/(lb+l0+l1).sum():.3f}")
print(f"gathered keys: seg={ (lb+l0+l1).sum() }  pair-design={ (2*lb+l0+l1).sum() }  per-block sum={nnz}")
print(f"tile-chunks executed: seg={(2*ch(lb)+ch(l0)+ch(l1)).sum()}  pair-design={(ch(lb+l0)+ch(lb+l1)).sum()}  quad-union={(2*ch(lb+l0+l1)).sum()}")
print(f"chunks gathered: seg={(ch(lb)+ch(l0)+ch(l1)).sum()} pair={(ch(lb+l0)+ch(lb+l1)).sum()}")
m = np.minimum(ch(l0), ch(l1))
tail = np.abs(ch(l0) - ch(l1))
print(f"128-key chunks: shared={ch(lb).sum()} interleaved-pairs={2*m.sum()} single-tile tail={tail.sum()}")
# 64-key chunk accounting for the double-buffered kernel (tile-chunk = 128 rows x 64 keys)
tc64 = (2 * ch64(lb) + ch64(l0) + ch64(l1)).sum()
g64 = (ch64(lb) + ch64(l0) + ch64(l1)).sum()
useful_rows_keys = nnz * 64
print(f"64-key: tile-chunks={tc64} chunks gathered={g64} useful fraction of tile-chunk work={useful_rows_keys / (tc64 * 128 * 64):.3f}")
