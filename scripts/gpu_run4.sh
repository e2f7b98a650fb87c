python -m pytest tests/test_gpu_slice.py tests/test_gpu_parity.py -k "slice or c4 or iteration or errors or rerun or store_paths" -x -q > gpurun_out/slice.log 2>&1; tail -15 gpurun_out/slice.log
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 2500 gpurun_out/bench_c4.json; tail -5 gpurun_out/bench_c4.err
LOBSTER_LOG=2 timeout 300 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/bench_c4_log2.err; tail -25 gpurun_out/bench_c4_log2.err
