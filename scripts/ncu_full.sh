# full ncu capture of one launch of a kernel (regex): ncu_full.sh KERNEL SKIP TAG [CONFIG]
# CONFIG: a bench.py config (C1..C5) run through profile_cfg.py; default C2 max-mult (profile_c2.py)
set -x
mkdir -p gpurun_out
K=${1:-join_write}
S=${2:-60}
TAG=${3:-direct}
CFG=${4:-}
if [ -z "$CFG" ]; then CMD="python scripts/profile_c2.py 3"; else CMD="python scripts/profile_cfg.py $CFG 1"; fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
