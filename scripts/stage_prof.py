"""One vecattn_forward at dit128k (VIDEO, ALG1) for an ncu launch list of its kernels."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
wl = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "dit128k"]
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0039
dev = torch.device("cuda")
q, k, v = bench.build_inputs(wl, "video", dev, 0, wl.Hq)
cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=alpha)
for _ in range(2):
    o, lse, off, idx = va.forward(q, k, v, cfg, causal=wl.causal)
torch.cuda.synchronize()
