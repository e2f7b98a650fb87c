set -x
mkdir -p gpurun_out
for r in 1 2; do LOBSTER_FJ_R=$r timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_r$r.json 2>gpurun_out/ab_r$r.err; python -c "
import json; d=json.load(open('gpurun_out/ab_r$r.json')); r=d['roofline']; print('R=$r', 'ms %.2f'%d['ms_per_step'], 'fj_us %.1f'%r['avg_launch_us'], 'frac %.3f'%r['frac'], d['phases_ms'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python scripts/profile_cfg.py C2 1 > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_C2.csv 14
