"""Summarise an ncu --csv launch list (gpu__time_duration per kernel)."""
import csv, collections, statistics as st, sys
rows = list(csv.reader(open(sys.argv[1])))
frames = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = None; data = collections.defaultdict(lambda: collections.defaultdict(list)); order = []
for r in rows:
    if not r: continue
    if r[0] == "ID": hdr = r; continue
    if hdr is None or len(r) < len(hdr): continue
    d = dict(zip(hdr, r)); name = d["Kernel Name"].split("(")[0][:48]
    if name not in order: order.append(name)
    data[name][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
tot = 0.0
for k in order:
    t = data[k]["gpu__time_duration.sum"]
    per_frame = sum(t) / frames / 1000
    tot += per_frame
    print(f"{k:48s} launches={len(t):4d} median_us={st.median(t)/1000:8.2f} per_frame_us={per_frame:8.2f}")
print(f"total per frame (serialised) = {tot:.1f} us")
