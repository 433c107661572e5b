"""Summarise ncu outputs into profiles/: launch-list shares + key --set full metrics.
usage: python scripts/summarize_ncu.py TAG   (reads gpurun_out/launches_TAG.csv, prof_TAG.ncu-rep)"""
import csv, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)
lines = [f"# ncu summary {tag}", ""]

lf = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
if os.path.exists(lf):
    rows = list(csv.reader(open(lf)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = {}
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            agg.setdefault(r[ki], []).append(float(r[vi].replace(",", "")) / 1e6)
    ours = {k: v for k, v in agg.items() if "va::" in k or "attn_" in k or "select_kernel" in k}
    lines += ["## Launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)", "",
              "Source command: `ncu --metrics gpu__time_duration.sum --clock-control none --csv "
              "python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --alpha 1.0039 --dense-reps 1 --no-context --no-causal-extra`", "",
              "| kernel | launches | mean ms | total ms |", "|---|---|---|---|"]
    for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k[:70]}` | {len(v)} | {sum(v)/len(v):.3f} | {sum(v):.2f} |")
    # share of one select+sparse step (pool, select, scan, emit, worklist, sparse attn)
    def mean(sub):
        xs = [x for k, v in ours.items() if sub in k for x in v]
        return sum(xs) / len(xs) if xs else 0.0
    # one vecattn_forward step (the bench's timed call): pool, select, scan, emit (CSR), plan, attention
    step = {n: mean(n) for n in ["pool_kernel", "select_kernel", "scan_kernel", "emit_kernel", "plan_kernel"]}
    sp = [x for k, v in ours.items() if "attn_db_kernel<128" in k or "attn_kernel<128, 1>" in k or "attn_kernel<128, true>" in k
          for x in v]
    step["attn_kernel<gather>"] = sum(sp) / len(sp) if sp else 0.0
    tot = sum(step.values())
    lines += ["", "Per-step shares (one vecattn_forward call = the bench step):", "", "| stage | ms | share |", "|---|---|---|"]
    for n, t in step.items():
        lines.append(f"| {n} | {t:.3f} | {100*t/tot:.1f}% |")
    lines.append(f"| total | {tot:.3f} | 100% |")

rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
summary = {}
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "launch__block_size"]
    lines += ["", "## --set full (one launch; full bench workload, 24 heads, vecattn_forward)", ""]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        d = {}
        for w in want:
            if w in h:
                d[w] = f"{r[h.index(w)]} {units[h.index(w)]}".strip()
        summary[name] = d
        lines += [f"### `{name}`", ""] + [f"- {k}: {v}" for k, v in d.items()] + [""]
open(os.path.join(out_dir, f"ncu_{tag}.md"), "w").write("\n".join(lines) + "\n")
# per-launch DRAM traffic of the sparse attention kernel (bench.py roofline.traffic)
for name, d in summary.items():
    if "attn_db_kernel<128" in name or "attn_kernel<128, 1>" in name or "attn_kernel<128, true>" in name:
        def num(x):
            v, u = x.split()[0], x.split()[1] if len(x.split()) > 1 else ""
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
            return float(v) * mult
        tr = num(d["dram__bytes_read.sum"]) + num(d["dram__bytes_write.sum"])
        json.dump({"kernel": name, "dram_bytes_per_launch": tr, "source": f"profiles/ncu_{tag}.md",
                   "workload": "dit128k, 24 heads, vecattn_forward"},
                  open(os.path.join(out_dir, "traffic.json"), "w"), indent=1)
json.dump(summary, open(os.path.join(out_dir, f"ncu_{tag}.json"), "w"), indent=1)
print("\n".join(lines))
