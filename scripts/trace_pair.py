"""Timeline of the CTA-pair sparse attention kernel (VECATTN_TRACE debug hook): %globaltimer
(ns) per chunk in the leader (blockIdx 0) and the peer (blockIdx 1, kinds + 16), as recorded in
csrc/attn_pair.cu.  dit128k VIDEO, 2 heads, ALG1 at rho ~ 0.785."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
os.environ["VECATTN_PAIR"] = "1"
dev = torch.device("cuda")
wl = synth.WORKLOADS["dit128k"]
q, k, v = bench.build_inputs(wl, "video", dev, 0, 2)
cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=1.0039)
off, idx = va.select(q, k, cfg)
tr = torch.zeros(32 * 4096, dtype=torch.int64, device=dev)
va.sparse_fwd(q, k, v, off, idx, pq=64)
torch.cuda.synchronize()
os.environ["VECATTN_TRACE"] = str(tr.data_ptr())
va.sparse_fwd(q, k, v, off, idx, pq=64)
torch.cuda.synchronize()
t = tr.view(32, 4096).cpu().numpy().astype(np.int64)
# kinds: 0 K issue (loader), 10 K issued, 11 V issued, 2 K landed (MMA), 12 S issued, 6/8 S ready (WG0/WG1 q0),
# 7/9 P done (q0), 15 last softmax warp's P, 5 P seen (MMA), 4 PV issued
n = int((t[4] > 0).sum())
t0 = t[t > 0].min()
print("chunks traced:", n)
def st(x): return f"median {np.median(x):.0f} p10 {np.percentile(x, 10):.0f} p90 {np.percentile(x, 90):.0f} (n={len(x)})" if len(x) else "n/a"
def d(a, b):
    return np.array([t[b, c] - t[a, c] for c in range(4, n - 4) if t[a, c] > 0 and t[b, c] > 0])
sready = np.where(t[6] > 0, t[6], t[8]); pdone = np.where(t[7] > 0, t[7], t[9])
last = np.maximum(t[15], t[31])
rows = []
for c in range(4, n - 4):
    if sready[c] > 0 and pdone[c] > 0 and t[5, c] > 0:
        rows.append((t[12, c] - t[2, c], sready[c] - t[12, c], pdone[c] - sready[c], last[c] - pdone[c],
                     t[5, c] - last[c], t[4, c] - t[5, c]))
rows = np.array(rows)
for i, lab in enumerate(["K landed -> S issued", "S issued -> S ready (leader q0)", "softmax (leader q0)",
                         "leader q0 P -> last warp P (both CTAs)", "last warp P -> P seen (MMA)", "P seen -> PV issued"]):
    print(f"{lab:40s}", st(rows[:, i]))
for a, b, lab in [(0, 10, "K issue duration"), (0, 2, "K issue -> landed(seen)"), (12, 4, "S issued -> PV issued")]:
    print(f"{lab:40s}", st(d(a, b)))
w = np.array([t[31, c] - t[15, c] for c in range(4, n - 4) if t[15, c] > 0 and t[31, c] > 0])
print(f"{'peer last warp - leader last warp':40s}", st(w))
for e, lab in [(12, "S issue"), (4, "PV issue")]:
    x = np.array([t[e, c] for c in range(n) if t[e, c] > 0])
    print(f"period {lab:33s}", st(np.diff(x)))
print("chunk: K landed / S issued / S ready / P q0 / last P / P seen / PV issued (ns)")
for c in list(range(0, 8)) + list(range(300, 306)):
    print(c, [int(v - t0) if v > 0 else -1 for v in (t[2, c], t[12, c], sready[c], pdone[c], last[c], t[5, c], t[4, c])])
