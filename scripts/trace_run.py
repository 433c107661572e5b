"""Timeline of CTA 0 of the sparse attention kernel (VECATTN_TRACE debug hook)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
mode = sys.argv[1] if len(sys.argv) > 1 else "video"
dev = torch.device("cuda")
if mode == "video":
    wl = synth.WORKLOADS["dit128k"]
    q, k, v = bench.build_inputs(wl, "video", dev, 0, 2)
    cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=1.0039)
    off, idx = va.select(q, k, cfg)
else:
    N, H, D = 32768, 8, 128
    q = torch.randn(1, H, N, D, device=dev).bfloat16(); k = torch.randn_like(q); v = torch.randn_like(q)
    sel = torch.arange(0, N, 2, device=dev)
    idx = sel.int().repeat(H * N // 64)
    off = torch.arange(0, H * N // 64 + 1, device=dev, dtype=torch.int64) * sel.numel()
tr = torch.zeros(32 * 4096, dtype=torch.int64, device=dev)
va.sparse_fwd(q, k, v, off, idx, pq=64)
torch.cuda.synchronize()
os.environ["VECATTN_TRACE"] = str(tr.data_ptr())
va.sparse_fwd(q, k, v, off, idx, pq=64)
torch.cuda.synchronize()
t = tr.view(32, 4096).cpu().numpy().astype(np.int64)
n = int((t[2] > 0).sum())
t0 = t[t > 0].min()
names = ["K_issue", "V_issue", "K_landed", "V_landed", "PV0_issued", "PV1_issued", "S0_ready", "P0_done", "S1_ready", "P1_done"]
print("chunks traced:", n)
for c in list(range(0, 12)) + list(range(100, 106)):
    row = " ".join(f"{names[e]}={(t[e, c] - t0) if t[e, c] > 0 else -1:9d}" for e in range(10))
    print(c, row)
d = lambda a, b: np.array([t[b, c] - t[a, c] for c in range(2, n - 2) if t[a, c] > 0 and t[b, c] > 0])
def st(x): return f"median {np.median(x):.0f} p90 {np.percentile(x, 90):.0f} (n={len(x)})" if len(x) else "n/a"
print("K gather latency (K_issue->K_landed):", st(d(0, 2)))
print("V gather latency (V_issue->V_landed):", st(d(1, 3)))
print("softmax0 (S0_ready->P0_done):", st(d(6, 7)))
print("softmax1 (S1_ready->P1_done):", st(d(8, 9)))
per = np.diff(np.array([t[2, c] for c in range(n)]))
print("  tile0 P0_done->PV0_issued:", st(d(7, 4)))
print("  V_landed->PV0_issued:", st(d(3, 4)))
print("chunk period (K_landed[c+1]-K_landed[c]):", st(per))
issue = np.diff(np.array([t[0, c] for c in range(n)]))
print("K issue period:", st(issue))
print("K issue duration (K_issue->K_issue_end):", st(d(0, 10)))
print("V issue duration (V_issue->V_issue_end):", st(d(1, 11)))
print("K issue_end->landed:", st(d(10, 2)))
print("V issue_end->landed:", st(d(11, 3)))
# item boundaries: the largest gaps between consecutive S0_ready events
s0 = np.array([t[6, c] for c in range(n) if t[6, c] > 0])
g = np.diff(s0)
print("S0_ready period:", st(g))
print("largest S0_ready gaps (ns, item boundaries):", np.sort(g)[-8:].tolist())
