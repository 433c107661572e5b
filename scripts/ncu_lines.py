"""Aggregate ncu warp-stall samples per CUDA source line (cuda,sass source page CSV).
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > f.csv; python ncu_lines.py f.csv [N]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = collections.Counter(); stalls = collections.defaultdict(collections.Counter); text = {}
cur_file = None; h = None; line = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": h = r; continue
    if h is None or len(r) < 5: continue
    if r[0].strip():
        line = (cur_file, int(r[0])); text[line] = r[1].strip()
    try: s = float(r[4] or 0)
    except ValueError: continue
    agg[line] += s
    for i, name in enumerate(h):
        if name.startswith("stall_") and "Not Issued" not in name and i < len(r):
            try: v = float(r[i] or 0)
            except ValueError: continue
            if v: stalls[line][name[6:]] += v
tot = sum(agg.values())
print("total samples", tot)
for k, v in agg.most_common(n_top):
    top = ", ".join(f"{a}:{100*b/v:.0f}%" for a, b in stalls[k].most_common(3))
    print(f"{k[0]}:{k[1]:4d} {100*v/tot:5.1f}%  {text.get(k,'')[:70]:70s} [{top}]")
