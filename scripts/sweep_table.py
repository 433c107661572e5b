"""Render gpurun_out/sweep_TAG.jsonl (scripts/sweep.sh) as profiles/sweep_TAG.md."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = [json.loads(l) for l in open(os.path.join(ROOT, "gpurun_out", f"sweep_{tag}.jsonl")) if l.strip().startswith("{")]
out = [f"# Sweep {tag} (1xB200, kernel-only bench lines; `scripts/sweep.sh`)", "",
       "Each line is `bench.py --no-e2e --no-cpu-baseline --steps 3` on the named workload (VIDEO inputs unless noted),",
       "alpha calibrated by bisection to the target sparsity (MINS_ALG1 unless noted). `fwd` = one vecattn_forward",
       "(pool, select, scan, CSR emit, plan, attention); speed-up = dense / fwd; attention TFLOP/s = useful",
       "4*D*sum|J_r| flops / attention-kernel time; select GB/s = algorithmic bytes / (pool+select+scan) time.", "",
       "| workload | kind | mode | causal | H/Hkv | N | P_q | B_K | G_K | rho | fwd ms | select ms | plan ms | attn ms | dense ms | speed-up | attn TFLOP/s (frac) | dense TFLOP/s | select GB/s | SM MHz |",
       "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
for d in rows:
    c = d["config"]; st = d.get("stage_ms", {}); sr = d.get("select_roofline", {})
    kind = "gauss" if "GAUSS" in d.get("data", "") else "video"
    out.append(f"| {c['workload']} | {kind} | {c['mode']} | {c['causal']} | {c['H']}/{c['Hkv']} | {c['N']} | "
               f"{c['pq']} | {c['bk']} | {c['gk']} | "
               f"{c['rho_achieved']:.3f} | {d['forward_ms']:.2f} | {st.get('select', -1):.2f} | {st.get('emit_plan', -1):.2f} | "
               f"{st.get('attention', -1):.2f} | {(d['dense_ms'] or float('nan')):.1f} | {(d['speedup_vs_dense'] or float('nan')):.2f} | "
               f"{d['roofline']['achieved']:.0f} ({d['roofline']['frac']:.2f}) | {(d['dense_tflops'] or float('nan')):.0f} | "
               f"{sr.get('achieved', 0):.0f} | {(d['clocks']['sm_mhz'] or float('nan')):.0f} |")
open(os.path.join(ROOT, "profiles", f"sweep_{tag}.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
