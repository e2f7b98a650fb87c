"""Brief summary of an ncu report (first kernel): key details + top stall reasons.
usage: python scripts/ncu_brief.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ('Duration', 'Registers Per Thread', 'Achieved Occupancy', 'Warp Cycles Per Issued Instruction',
        'Issue Slots Busy', 'Avg. Active Threads Per Warp', 'Avg. Not Predicated Off Threads Per Warp',
        'Compute (SM) Throughput', 'L1/TEX Hit Rate', 'Executed Ipc Active', 'Block Size', 'Grid Size',
        'Dynamic Shared Memory Per Block', 'Memory Throughput', 'DRAM Throughput', 'L2 Hit Rate')
r = csv.reader(io.StringIO(det))
h = next(r)
name = None
for row in r:
    d = dict(zip(h, row))
    name = name or d.get('Kernel Name')
    if d['Metric Name'] in want:
        print(f"{d['Metric Name']}: {d['Metric Value']} {d['Metric Unit']}")
print("kernel:", name)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(raw))
h = next(r); next(r); v = next(r)
d = dict(zip(h, v))
st = [(k, float(x)) for k, x in d.items()
      if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')]
for k, x in sorted(st, key=lambda t: -t[1])[:8]:
    print(f"stall {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}: {x:.2f}")
for k in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__inst_executed.sum', 'smsp__thread_inst_executed_per_inst_executed.ratio'):
    if k in d:
        print(k, d[k])
