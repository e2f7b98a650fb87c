set -x
python -m pytest tests/test_gpu_shards.py -x -q --durations=5 > gpurun_out/shards.log 2>&1; tail -5 gpurun_out/shards.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_overlap.json 2> gpurun_out/bench_overlap.err; tail -c 3000 gpurun_out/bench_overlap.json; tail -5 gpurun_out/bench_overlap.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --serial > gpurun_out/bench_serial.json 2>&1; tail -c 1500 gpurun_out/bench_serial.json
LOBSTER_LOG=2 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --serial --no-e2e > gpurun_out/bench_log2.json 2> gpurun_out/bench_log2.err; tail -3 gpurun_out/bench_log2.err
