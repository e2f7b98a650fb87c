python -m pytest tests/test_gpu_parity.py tests/test_gpu_dmaxmin.py -x -q -k "c1 or random or c2_reduced or c5_reduced or mutual or store_paths or determinism or c2_full" > gpurun_out/fast32_tests.log 2>&1; tail -3 gpurun_out/fast32_tests.log
for f in 1 0 1 0; do
LOBSTER_FAST32=$f timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --serial > gpurun_out/b_f$f.json 2>&1
python - <<PY
import json; d=json.loads(open('gpurun_out/b_f$f.json').read().strip().splitlines()[-1])
print('fast32=$f', round(d['ms_per_step'],2), 'frac', round(d['roofline']['frac'],4), 'us/launch', round(d['roofline']['avg_launch_us'],1))
PY
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_overlap.json 2>&1; tail -c 600 gpurun_out/b_overlap.json
