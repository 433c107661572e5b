"""Selection time for one rank's share of heads (few rows): vlm64k with 4 of 28 heads."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
for wl_name, h1, alpha in (("vlm64k", 4, 0.39), ("vlm64k", 28, 0.39), ("dit128k", 24, 1.0039)):
    wl = synth.WORKLOADS[wl_name]
    q, k, v = bench.build_inputs(wl, "video", torch.device("cuda"), 0, h1)
    cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=alpha)
    ws = va.Workspace("cuda")
    for _ in range(2): va.select(q, k, cfg, causal=wl.causal, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): va.select(q, k, cfg, causal=wl.causal, ws=ws)
    e1.record(); torch.cuda.synchronize()
    print(wl_name, h1, "heads:", f"{e0.elapsed_time(e1)/5:.3f} ms per select")
