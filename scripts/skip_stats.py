"""How many softmax exponentials the sparse attention kernel computes for non-member rows,
and how many a warp-uniform skip would save.

A warp of the softmax covers 32 rows of one P_q = 64 block, so for every key of a chunk the
whole warp is either a member or not.  For each item (4 blocks, tiles (01|23)) this counts
  * computed: tile-chunks x 64 keys x 128 rows (the kernel today);
  * useful:   sum of block sizes x 64 rows;
  * skipped:  16-key column groups in which a warp's block has no member, when the keys of
              each plan segment are ordered by their membership pattern (ORDER below) --
              per warp, 16 columns x 32 rows each.
Usage: python scripts/skip_stats.py [workload] [heads] [alpha]
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
GW = int(os.environ.get("GW", "16"))
dev = torch.device("cuda")
q, k, v = bench.build_inputs(wl, "video", dev, 0, H)
cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=alpha)
off, idx = va.select(q, k, cfg, causal=wl.causal)
torch.cuda.synchronize()
N = wl.N
Np = (N + 63) // 64
ch = lambda x: (x + 63) // 64

# pattern rank: both-segment by (b0b1 in order 1,3,2) major, (b2b3 in order 1,3,2) minor
o3 = {1: 0, 3: 1, 2: 2}
rank = np.full(16, 99, dtype=np.int64)
for p in range(1, 16):
    lo, hi = p & 3, p >> 2
    if lo and hi:
        rank[p] = o3[lo] * 3 + o3[hi]
    elif lo:
        rank[p] = 10 + o3[lo]
    else:
        rank[p] = 20 + o3[hi]
rank_t = torch.tensor(rank, device=dev)

computed = useful = kept_sorted = kept_keyorder = 0
offc = off.cpu()
for h in range(H):
    for it in range(Np // 4):
        r0 = h * Np + 4 * it
        a, b = int(offc[r0]), int(offc[r0 + 4])
        ids = idx[a:b].long()
        bl = torch.repeat_interleave(torch.arange(4, device=dev), (offc[r0 + 1:r0 + 5] - offc[r0:r0 + 4]).to(dev))
        pat = torch.zeros(N, dtype=torch.int64, device=dev)
        pat.index_put_((ids,), (1 << bl), accumulate=True)
        useful += (b - a) * 64
        keys = torch.nonzero(pat).squeeze(1)
        pk = pat[keys]
        for sort in (False, True):
            pp = pk[torch.argsort(rank_t[pk] * (1 << 20) + keys)] if sort else pk[torch.argsort((rank_t[pk] // 10) * (1 << 20) + keys)]
            r = rank_t[pp]
            segs = [pp[r < 10], pp[(r >= 10) & (r < 20)], pp[r >= 20]]
            kept = 0
            comp = 0
            for t in range(2):
                for s in (segs[0], segs[1 + t]):
                    n = s.numel()
                    if n == 0:
                        continue
                    padded = torch.zeros(ch(n) * 64, dtype=torch.int64, device=dev)
                    padded[:n] = s
                    comp += ch(n) * 64 * 128
                    g = padded.view(-1, GW)
                    for bb in (2 * t, 2 * t + 1):
                        live = ((g >> bb) & 1).any(dim=1)
                        kept += int(live.sum()) * GW * 64
            if sort:
                kept_sorted += kept
            else:
                kept_keyorder += kept
                computed += comp
print(f"workload {wl.name if hasattr(wl, 'name') else sys.argv[1:2]} heads {H} group {GW}")
print(f"useful/computed      {useful / computed:.3f}")
print(f"kept/computed (key order, warp skip)     {kept_keyorder / computed:.3f}")
print(f"kept/computed (pattern order, warp skip) {kept_sorted / computed:.3f}")
