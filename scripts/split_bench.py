import os, sys, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
wl = synth.WORKLOADS["dit128k"]
q, k, v = bench.build_inputs(wl, "video", torch.device("cuda"), 0, 3)   # one rank's share at 8 GPUs
cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=1.0039)
ws = va.Workspace("cuda")
for n in ("1", "auto"):
    if n == "auto": os.environ.pop("VECATTN_SELECT_SPLIT", None)
    else: os.environ["VECATTN_SELECT_SPLIT"] = n
    for _ in range(2): va.select(q, k, cfg, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): va.select(q, k, cfg, ws=ws)
    e1.record(); torch.cuda.synchronize()
    print("3 heads, split", n, f"{e0.elapsed_time(e1)/5:.3f} ms per select (incl. host sync for capacity)")
