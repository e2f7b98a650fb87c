# bench one config quickly + ncu full capture of its first launch of kernel regex $2
set -x
mkdir -p gpurun_out
c=${1:-C3}; k=${2:-tile_fixpoint}
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; cut -c1-300 gpurun_out/bench_$c.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/prof_$c python scripts/profile_cfg.py $c 1 > gpurun_out/ncu_$c.log 2>&1; tail -2 gpurun_out/ncu_$c.log
