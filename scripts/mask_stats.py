"""How many tile-chunks of the sparse plan need the block-membership mask (keys of the
tile's union that miss one of its two P_q=64 blocks)?  Ascending order vs grouped by
membership pattern.  dit128k VIDEO, 2 heads, 64-key chunks."""
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
tot = need_asc = need_grp = 0
for h in range(2):
    for it in range(Np // 4):
        r0 = h * Np + 4 * it
        mem = {}
        for b in range(4):
            for key in ih[oh[r0 + b]:oh[r0 + b + 1]]:
                mem[key] = mem.get(key, 0) | (1 << b)
        keys = np.array(sorted(mem)); bits = np.array([mem[x] for x in keys])
        t0 = (bits & 3) != 0; t1 = (bits & 12) != 0
        full0 = (bits & 3) == 3; full1 = (bits & 12) == 12
        segs = [(t0 & t1), (t0 & ~t1), (t1 & ~t0)]
        for t, (inT, fullT) in enumerate(((t0, full0), (t1, full1))):
            for sg in segs:
                sel = sg & inT
                if not sel.any():
                    continue
                f = fullT[sel]
                n = f.size
                ch = (n + 63) // 64
                tot += ch
                need_asc += sum(1 for c in range(ch) if not f[64 * c:64 * c + 64].all())
                fs = np.sort(~f)  # full (False) first
                need_grp += sum(1 for c in range(ch) if fs[64 * c:64 * c + 64].any())
print(f"tile-chunks {tot}: need mask ascending {need_asc} ({100*need_asc/tot:.1f}%), grouped {need_grp} ({100*need_grp/tot:.1f}%)")
