# usage: bash scripts/prof_c3c4.sh [configs...]  — LOBSTER_LOG trace + launch list per config
set -x
mkdir -p gpurun_out
for c in "${@:-C3 C4}"; do
LOBSTER_LOG=1 python scripts/profile_cfg.py $c 3 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python scripts/profile_cfg.py $c 1 > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_$c.csv 12
done
