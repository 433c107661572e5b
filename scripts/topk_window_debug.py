"""Windowed-TOPK diagnostics over several workloads and keep fractions: VECATTN_TOPK_DEBUG makes
the library print, per selection, the rows whose window missed (radix fallback), candidate-slice
overflows, the mean / max candidates per row and a hash of every row's window bounds."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, torch
sys.path.insert(0, "%s")
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
cases = [("dit128k", 24, 0.215, False), ("dit128k", 6, 0.01, False), ("dit128k", 6, 0.9, False),
         ("vlm128k", 28, 0.215, True), ("hy", 8, 0.3, False), ("dit16k", 4, 0.5, False), ("wan", 8, 0.1, False)]
for name, H, f, causal in cases:
    wl = synth.WORKLOADS[name]
    q, k, _ = bench.build_inputs(wl, "video", torch.device("cuda"), 0, H)
    print(name, H, f, causal, file=sys.stderr, flush=True)
    va.select(q, k, va.SelectConfig(mode="topk", pq=64, keep_frac=f), causal=causal)
    torch.cuda.synchronize()
    del q, k
''' % ROOT
env = dict(os.environ, VECATTN_TOPK_DEBUG="1")
out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
for l in out.stderr.splitlines():
    if "[topk window]" in l or l.split(" ")[0] in ("dit128k", "vlm128k", "hy", "dit16k", "wan") or "Error" in l:
        print(l)
