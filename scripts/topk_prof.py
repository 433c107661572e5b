import os, sys, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
wl = synth.WORKLOADS["dit128k"]
q, k, v = bench.build_inputs(wl, "video", torch.device("cuda"), 0, 4)
cfg = va.SelectConfig(mode="topk", pq=64, keep_frac=0.215)
off, idx = va.select(q, k, cfg)
torch.cuda.synchronize()
print("nnz", int(off[-1]))
