"""gpurun_out/traffic.csv (ncu metrics-only pass over every launch of the dominant
kernel) -> profiles/ncu_traffic.json: average DRAM bytes and duration per launch."""
import csv, json, sys
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/traffic.csv")))
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        h = rows[i]; data = rows[i + 1:]; break
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
per = {}
for r in data:
    if len(r) <= vi:
        continue
    key = (r[0], r[ki])
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "nsecond": 1e-3, "ms": 1e3}.get(u, 1)
    per.setdefault(key, {})[r[mi]] = v * scale
launches = list(per.values())
n = len(launches)
rd = sum(l.get("dram__bytes_read.sum", 0) for l in launches) / n
wr = sum(l.get("dram__bytes_write.sum", 0) for l in launches) / n
t = sum(l.get("gpu__time_duration.sum", 0) for l in launches) / n
name = list(per.keys())[0][1].split("(")[0]
out = {"kernel": name, "launches": n, "dram_read_bytes_per_launch": rd, "dram_write_bytes_per_launch": wr,
       "dram_bytes_per_launch": rd + wr, "avg_duration_us_ncu": t,
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum over every launch "
                 "of the kernel in one C2 run (max-mult + max-min), scripts/ncu_traffic.sh"}
json.dump(out, open(sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
