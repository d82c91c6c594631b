"""Like ncu_lines.py, sorted by instructions executed (the issue-bound view)."""
import csv, sys, collections
path = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
hdr = None; src = {}; stats = collections.defaultdict(lambda: [0, 0])
cur_line = None
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8:
        continue
    line, code = r[0], r[1]
    if line:
        cur_line = int(line); src[cur_line] = code
    try:
        samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        inst = float(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    if cur_line is not None:
        stats[cur_line][0] += samp; stats[cur_line][1] += inst
tot_s = sum(v[0] for v in stats.values()) or 1; tot_i = sum(v[1] for v in stats.values()) or 1
print(f"total instructions {tot_i:.4g}")
for ln, (s, i) in sorted(stats.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{ln:5d} inst={100*i/tot_i:5.1f}% stall={100*s/tot_s:5.1f}%  {src.get(ln,'')[:110]}")
