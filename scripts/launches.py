"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv')))
for i, r in enumerate(rows):
    if r and r[0] == 'ID':
        hdr = r; start = i + 1; break
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[start:]:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0].replace('void ', '').replace('lob::', '').replace('(anonymous namespace)::', '').replace('<unnamed>::', '')
    v = float(r[vi].replace(',', ''))
    v = v / 1e6 if r[ui] in ('nsecond', 'ns') else (v / 1e3 if r[ui] in ('usecond', 'us') else v)
    agg[name][0] += 1; agg[name][1] += v
tot = sum(a[1] for a in agg.values())
print(f"{'ms':>9} {'share':>6} {'launches':>8} {'avg_us':>9}  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{t:9.2f} {100*t/tot:5.1f}% {n:8d} {1000*t/n:9.1f}  {k}")
print(f"total {tot:.2f} ms over {sum(a[0] for a in agg.values())} launches")
