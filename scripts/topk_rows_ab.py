"""Window bounds of the windowed TOPK from the warp-per-row tk_rows stages vs the thread-per-row
walk (VECATTN_TK_ROWS_THREAD=1): VECATTN_TOPK_DEBUG prints a hash of every row's [lo, hi]."""
import os, subprocess, sys
code = r'''
import os, sys, torch
sys.path.insert(0, "%s")
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
for name, H, f, causal in (("dit128k", 6, 0.215, False), ("vlm128k", 8, 0.1, True), ("dit16k", 4, 0.5, False)):
    wl = synth.WORKLOADS[name]
    q, k, _ = bench.build_inputs(wl, "video", torch.device("cuda"), 0, H)
    va.select(q, k, va.SelectConfig(mode="topk", pq=64, keep_frac=f), causal=causal)
    torch.cuda.synchronize()
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for thread in (False, True):
    env = dict(os.environ, VECATTN_TOPK_DEBUG="1")
    if thread:
        env["VECATTN_TK_ROWS_THREAD"] = "1"
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("thread" if thread else "warp  ", [l for l in out.stderr.splitlines() if "[topk window]" in l])
