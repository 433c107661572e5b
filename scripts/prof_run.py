"""Minimal launch sequence for ncu: select, sparse, dense (x2) on a bench workload."""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="dit128k")
ap.add_argument("--kind", default="video")
ap.add_argument("--alpha", type=float, default=1.0039)
ap.add_argument("--heads", type=int, default=0, help="limit query heads (0 = all)")
ap.add_argument("--no-dense", action="store_true")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--fused", action="store_true", help="use vecattn_forward")
a = ap.parse_args()
wl = synth.WORKLOADS[a.workload]
dev = torch.device("cuda", 0)
h1 = a.heads or wl.Hq
q, k, v = bench.build_inputs(wl, a.kind, dev, 0, h1)
cfg = va.SelectConfig(mode="alg1", pq=64, bk=16, gk=wl.gk, alpha=a.alpha)
ws = va.Workspace(dev)
for _ in range(a.reps):
    if a.fused:
        o, lse, off, idx = va.forward(q, k, v, cfg, causal=wl.causal)
    else:
        off, idx = va.select(q, k, cfg, causal=wl.causal, ws=ws)
        o, lse = va.sparse_fwd(q, k, v, off, idx, pq=64, causal=wl.causal)
    if not a.no_dense:
        od, _ = va.dense_fwd(q, k, v, causal=wl.causal)
torch.cuda.synchronize()
print("nnz", int(off[-1]))
