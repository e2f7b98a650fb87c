# full ncu capture of one mid-fixpoint launch of a kernel (regex) in C2 max-mult
set -x
mkdir -p gpurun_out
K=${1:-join_write}
S=${2:-60}
TAG=${3:-direct}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/prof_$TAG python scripts/profile_c2.py 3 > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
