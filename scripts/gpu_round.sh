# usage: bash scripts/gpu_round.sh [tests] [bench] [ncu]
set -x
mkdir -p gpurun_out
for what in "$@"; do
case $what in
tests) timeout 1500 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15 ;;
quick) timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not full_size" 2>&1 | tail -15 ;;
smoke) python __graft_entry__.py --smoke 2>&1 | tail -3 ;;
bench) timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json ;;
prof) python scripts/profile_c2.py 3,1 2>&1 | tail -3 ;;
ncu) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_c2.py 3 > /dev/null 2>&1; wc -l gpurun_out/launches.csv ;;
configs) for c in C2 C1 C3 C4 C5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; cut -c1-400 gpurun_out/bench_$c.json; done ;;
esac
done
