"""Per-kernel time of one TOPK selection at dit128k (24 heads, keep 21.5%), via torch.profiler
(median over 3 profiled calls; kernels grouped by name and select epilogue)."""
import collections, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
from torch.profiler import ProfilerActivity, profile
H = int(sys.argv[1]) if len(sys.argv) > 1 else 24
wl = synth.WORKLOADS["dit128k"]
q, k, v = bench.build_inputs(wl, "video", torch.device("cuda"), 0, H)
cfg = va.SelectConfig(mode="topk", pq=64, keep_frac=0.215)
off, idx = va.select(q, k, cfg)
torch.cuda.synchronize()
runs = []
for _ in range(3):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        off, idx = va.select(q, k, cfg)
        torch.cuda.synchronize()
    agg = collections.OrderedDict()
    for e in prof.events():
        if e.device_type.name == "CUDA":
            agg[e.name[:90]] = agg.get(e.name[:90], 0.0) + e.device_time_total / 1000
    runs.append(agg)
tot = []
for name in runs[0]:
    ts = sorted(r.get(name, 0.0) for r in runs)
    print(f"{ts[1]:9.3f} ms  {name}")
if os.environ.get("TOPK_PROF_ALL"):  # every launch of the last profiled call, in order
    for e in prof.events():
        if e.device_type.name == "CUDA":
            print(f"   {e.device_time_total / 1000:9.3f} ms  {e.name[:70]}")
tot = sorted(sum(r.values()) for r in runs)
print(f"total {tot[1]:.3f} ms, nnz {int(off[-1])}")
