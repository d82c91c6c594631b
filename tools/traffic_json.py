"""Per-kernel DRAM traffic / duration summary of an ncu launch-list CSV
(`tools/ncu_launches.sh`): writes {kernel: {time_us, dram_read, dram_write,
launches}} medians per launch.  bench.py reads the committed copy
(profiles/r01_traffic.json) for the roofline `traffic` field."""
import csv, collections, json, statistics as st, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if not r: continue
    if r[0] == "ID": hdr = r; continue
    if hdr is None or len(r) < len(hdr): continue
    d = dict(zip(hdr, r)); name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("hs::", "")
    data[name][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
out = {}
for k, m in data.items():
    out[k] = {"launches": len(m["gpu__time_duration.sum"]),
              "time_us": st.median(m["gpu__time_duration.sum"]) / 1000.0,
              "dram_read_bytes": st.median(m.get("dram__bytes_read.sum", [0.0])),
              "dram_write_bytes": st.median(m.get("dram__bytes_write.sum", [0.0]))}
json.dump({"source": sys.argv[1], "note": "ncu --clock-control none, default cache control (caches flushed before each kernel): cold-cache per-launch numbers", "kernels": out}, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
