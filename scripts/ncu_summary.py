"""Key metrics + top stall reasons / SASS lines of an ncu --set full report.
usage: python scripts/ncu_summary.py REPORT.ncu-rep [--json OUT] [--top N]"""
import csv, io, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size", "smsp__inst_executed.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warp_latency_per_inst_issued.ratio", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 12
    r = ncu_csv(rep, "--page", "raw")
    h, units, v = r[0], r[1], r[2]
    res = {"Kernel Name": v[h.index("Kernel Name")][:120]}
    for k in KEYS:
        if k in h:
            res[k] = [v[h.index(k)], units[h.index(k)]]
    s = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    hh, rows = s[1], s[2:]
    si = hh.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(x[si] or 0) for x in rows) or 1.0
    res["sass_instructions"] = len(rows)
    stalls = {hh[i]: sum(float(x[i] or 0) for x in rows) / tot for i, n in enumerate(hh)
              if n.startswith("stall_") and "Not Issued" not in n}
    res["stall_share"] = {k: round(v, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
    res["top_sass"] = [f"{float(x[si]) / tot * 100:5.1f}% {x[1][:60]}"
                       for x in sorted(rows, key=lambda x: -float(x[si] or 0))[:top]]
    print(json.dumps(res, indent=1, ensure_ascii=False))
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1, ensure_ascii=False)


if __name__ == "__main__":
    main()
