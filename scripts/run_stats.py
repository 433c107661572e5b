"""Run-length statistics of the per-item key unions (4 blocks of 64 rows) on a bench workload:
how contiguous are the gathered K/V rows?"""
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
off, idx = va.select(q, k, va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=alpha), causal=wl.causal)
oh, ih = off.cpu().numpy(), idx.cpu().numpy()
Np = (wl.N + 63) // 64
runs_hist = np.zeros(20, np.int64)
keys_in_runs = np.zeros(20, np.int64)
tot_keys = 0; tot_runs = 0; chunk_contig = 0; chunks = 0; g4_contig = 0; g4 = 0
for h in range(H):
    for it in range(0, Np, 4):
        r0 = h * Np + it
        u = np.unique(ih[oh[r0]:oh[min(r0 + 4, (h + 1) * Np)]])
        if u.size == 0: continue
        brk = np.nonzero(np.diff(u) != 1)[0]
        starts = np.concatenate([[0], brk + 1]); ends = np.concatenate([brk + 1, [u.size]])
        L = ends - starts
        b = np.minimum(np.log2(L).astype(int), 19)
        np.add.at(runs_hist, b, 1); np.add.at(keys_in_runs, b, L)
        tot_keys += u.size; tot_runs += L.size
        for c0 in range(0, u.size, 64):
            c = u[c0:c0 + 64]; chunks += 1
            chunk_contig += int(c[-1] - c[0] == c.size - 1)
        n4 = u.size // 4
        g = u[:4 * n4].reshape(-1, 4)
        g4 += n4; g4_contig += int(((g[:, 3] - g[:, 0]) == 3).sum())
print(f"{wl.name}: union keys {tot_keys}, runs {tot_runs}, mean run {tot_keys/tot_runs:.1f}")
for i in range(20):
    if runs_hist[i]: print(f"  run len [{2**i},{2**(i+1)}): runs {runs_hist[i]}  keys {keys_in_runs[i]} ({100*keys_in_runs[i]/tot_keys:.1f}%)")
print(f"64-key chunks fully contiguous: {chunk_contig}/{chunks} ({100*chunk_contig/chunks:.1f}%)")
print(f"4-key groups contiguous: {g4_contig}/{g4} ({100*g4_contig/max(g4,1):.1f}%)")
