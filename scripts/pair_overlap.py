"""How much would sharing K/V gathers between adjacent 256-row items (2-CTA multicast) save?"""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
wl = synth.WORKLOADS["dit128k"]
q, k, v = bench.build_inputs(wl, "video", torch.device("cuda"), 0, 2)
off, idx = va.select(q, k, va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=1.0039))
oh, ih = off.cpu().numpy(), idx.cpu().numpy()
Np = wl.N // 64
tot_item = tot_pair = tot_quad = 0
for h in range(2):
    items = []
    for it in range(Np // 4):
        r0 = h * Np + 4 * it
        items.append(np.unique(ih[oh[r0]:oh[r0 + 4]]))
    for a in range(0, len(items), 2):
        u = np.union1d(items[a], items[a + 1])
        tot_item += items[a].size + items[a + 1].size
        tot_pair += u.size
    for a in range(0, len(items), 4):
        u = np.unique(np.concatenate(items[a:a + 4]))
        tot_quad += u.size
print(f"gathered keys: per item {tot_item}, per item-pair (2 CTAs) {tot_pair} ({tot_pair/tot_item:.3f}), "
      f"per 4 items {tot_quad} ({tot_quad/tot_item:.3f})")
