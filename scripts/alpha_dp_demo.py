"""NEXT-2 measurement: uniform alpha vs Eq. 4 per-head alphas (vecattn_alpha_dp) at the same
average sparsity, recall = fraction of each row's softmax mass kept (calibrate.py)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
from paper_2603_29494_b200 import calibrate as cal

rows = []
for wl_name, rho in (("dit32k", 0.785), ("dit32k", 0.9), ("vlm32k", 0.785)):
    wl = synth.WORKLOADS[wl_name]
    q, k, v = bench.build_inputs(wl, "video", torch.device("cuda"), 0, wl.Hq)
    cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk)
    a = cal.calibrate_uniform(q, k, cfg, rho, causal=wl.causal)
    lse_d = cal._dense_lse(q, k, v, wl.causal)
    sp_u, rec_u = cal.evaluate(q, k, v, cfg, wl.causal, lse_d, alpha=a)
    alphas = list(a * np.geomspace(0.2, 5.0, 25))
    prof = cal.profile_heads(q, k, v, alphas, cfg, causal=wl.causal)
    a_h, rec_pred, sp_pred = cal.per_head_alphas(prof, rho)
    sp_m, rec_m = cal.evaluate(q, k, v, cfg, wl.causal, lse_d, alpha_per_head=a_h)
    rows.append({"workload": wl_name, "rho_target": rho, "uniform_alpha": a, "uniform": [sp_u, rec_u],
                 "dp": [sp_m, rec_m], "alpha_per_head": a_h,
                 "head_sparsity_dp": [float(prof.sparsity[h, alphas.index(a_h[h])]) for h in range(wl.Hq)]})
    print(json.dumps(rows[-1]), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/alpha_dp_r01.json", "w"), indent=1)
