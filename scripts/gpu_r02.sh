# Round-2 GPU pass: tests, smoke, the C2 bench line, the ncu launch list of one
# C2 step, DRAM traffic of the dominant kernel, one full capture of a big round.
# usage: bash scripts/gpu_r02.sh [tests] [bench] [launches] [traffic] [full] [configs]
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for what in "$@"; do
case $what in
tests) timeout 2400 python -m pytest tests/ -x -q -m gpu --durations=15 > gpurun_out/gputests.log 2>&1; tail -25 gpurun_out/gputests.log ;;
smoke) timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -3 ;;
bench) timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json ;;
launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python scripts/profile_c2.py 1,3 > gpurun_out/launches_c2.log 2>&1; wc -l gpurun_out/launches_c2.csv ;;
traffic) timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:join_rows --csv --log-file gpurun_out/traffic.csv python scripts/profile_c2.py 1,3 > /dev/null 2>&1; wc -l gpurun_out/traffic.csv ;;
full) timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_rows -s 40 -c 1 -o gpurun_out/prof_join python scripts/profile_c2.py 3 > gpurun_out/ncu_join.log 2>&1; tail -2 gpurun_out/ncu_join.log ;;
configs) for c in C1 C3 C4 C5 C2P SG; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; cut -c1-300 gpurun_out/bench_$c.json; done ;;
newtests) timeout 1200 python -m pytest tests/test_gpu_tile.py tests/test_gpu_partition.py -x -q --durations=8 > gpurun_out/newtests.log 2>&1; tail -30 gpurun_out/newtests.log ;;
parity) timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; tail -8 gpurun_out/parity.log ;;
c3c1) for c in C1 C3; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; cut -c1-400 gpurun_out/bench_$c.json; done ;;
esac
done
