"""How much union waste a better block pairing inside a 256-row item would save.

For each item (4 consecutive P_q=64 blocks) compare the three ways to split it into two
128-row tiles: (01|23) (the kernel's), (02|13), (03|12).  Cost = 64-key tile-chunks of the
double-buffered kernel: 2*ch(|T0 & T1|) + ch(|T0 - T1|) + ch(|T1 - T0|).
"""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
wl = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "dit128k"]
H = int(sys.argv[2]) if len(sys.argv) > 2 else 2
alpha = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0039
dev = torch.device("cuda")
q, k, v = bench.build_inputs(wl, "video", dev, 0, H)
cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=alpha)
off, idx = va.select(q, k, cfg, causal=wl.causal)
torch.cuda.synchronize()
N = wl.N
Np = (N + 63) // 64
ch = lambda x: (x + 63) // 64
tot = np.zeros(4, dtype=np.int64)  # (01|23), (02|13), (03|12), best
useful = 0
offc = off.cpu()
for h in range(H):
    for it in range(Np // 4):
        r0 = h * Np + 4 * it
        a, b = int(offc[r0]), int(offc[r0 + 4])
        ids = idx[a:b].long()
        bl = torch.repeat_interleave(torch.arange(4, device=dev), (offc[r0 + 1:r0 + 5] - offc[r0:r0 + 4]).to(dev))
        m = torch.zeros(4, N, dtype=torch.bool, device=dev)
        m[bl, ids] = True
        useful += b - a
        costs = []
        for (x, y), (z, w) in (((0, 1), (2, 3)), ((0, 2), (1, 3)), ((0, 3), (1, 2))):
            t0 = m[x] | m[y]
            t1 = m[z] | m[w]
            lb = int((t0 & t1).sum()); l0 = int((t0 & ~t1).sum()); l1 = int((t1 & ~t0).sum())
            costs.append(2 * ch(lb) + ch(l0) + ch(l1))
        tot[:3] += costs
        tot[3] += min(costs)
print("tile-chunks (01|23) (02|13) (03|12) best:", tot.tolist())
print("useful fraction:", [useful * 64 / (t * 128 * 64) for t in tot])
