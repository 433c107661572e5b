"""Kernel-level A/B timing for the in-library attention kernels (one process per library
variant): dense dit128k (24 heads, N = 131072, non-causal) and the fused causal forward on
vlm64k (28/4 heads, ALG1 at a fixed alpha), L2 flushed, CUDA events, median of reps."""
import json, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
va.load()
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = {}

def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)

wl = synth.WORKLOADS["dit128k"]
q, k, v = bench.build_inputs(wl, "video", dev, 0, wl.Hq)
od = torch.empty_like(q); wsd = torch.empty(256, dtype=torch.uint8, device=dev)
if "dense" in sys.argv[1:] or len(sys.argv) == 1:
    out["dense_dit128k_ms"] = round(timed(lambda: va.dense_fwd_into(q, k, v, od, None, wsd, False)), 3)
if "sparse" in sys.argv[1:] or len(sys.argv) == 1:
    cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=1.0039)
    o, lse, off, idx = va.forward(q, k, v, cfg, causal=False)
    va.kernel_timing(True)
    ts = []
    for _ in range(3):
        flush.zero_(); va.forward(q, k, v, cfg, causal=False); torch.cuda.synchronize(); ts.append(va.kernel_timing_last()[2])
    va.kernel_timing(False)
    out["sparse_dit128k_attn_ms"] = round(statistics.median(ts), 3)
del q, k, v, od
wl = synth.WORKLOADS["vlm64k"]
q, k, v = bench.build_inputs(wl, "video", dev, 0, wl.Hq)
cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=0.4)
o, lse, off, idx = va.forward(q, k, v, cfg, causal=True)
va.kernel_timing(True)
ts = []
for _ in range(3):
    flush.zero_(); va.forward(q, k, v, cfg, causal=True); torch.cuda.synchronize(); ts.append(va.kernel_timing_last()[2])
va.kernel_timing(False)
out["causal_vlm64k_attn_ms"] = round(statistics.median(ts), 3)
print(json.dumps(out))
