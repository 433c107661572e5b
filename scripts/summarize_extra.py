"""Summarise the extra ncu captures (scripts/profile_extra.sh) into profiles/ncu_TAG_extra.md."""
import csv, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01f"
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
desc = {"select": "selection GEMM + Alg. 1 filter (select_kernel), dit128k, 24 heads",
        "dense": "dense attention (attn_kernel<128, dense>), dit128k, 4 heads",
        "causal": "causal sparse attention (attn_kernel<128, gather>), vlm128k, 28/4 heads"}
lines = [f"# ncu --set full, extra kernels ({tag}; `scripts/profile_extra.sh`)", ""]
for part in ("select", "dense", "causal"):
    rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}_{part}.ncu-rep")
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    lines += [f"## {part}: {desc[part]}", "", f"kernel: `{v[h.index('Kernel Name')][:90]}`", ""]
    for w in want:
        if w in h:
            lines.append(f"- {w}: {v[h.index(w)]} {u[h.index(w)]}".rstrip())
    if "dram__bytes_read.sum" in h:
        def num(i):
            x = float(v[i].replace(",", "")); un = u[i]
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(un, 1)
        t = float(v[h.index("gpu__time_duration.sum")].replace(",", "")) * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(u[h.index("gpu__time_duration.sum")], 1e-3)
        by = num(h.index("dram__bytes_read.sum")) + num(h.index("dram__bytes_write.sum"))
        lines.append(f"- achieved DRAM: {by / t / 1e9:.0f} GB/s ({by / 1e9:.2f} GB in {t * 1e3:.3f} ms)"
                     f" = {by / t / 1e9 / 6650:.2f} of 6650 GB/s (fallback), {by / t / 1e9 / 8000:.2f} of 8 TB/s nominal")
    lines.append("")
open(os.path.join(ROOT, "profiles", f"ncu_{tag}_extra.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
