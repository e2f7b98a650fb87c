# A/B of the stale slot read: relaxed GPU-scope load vs plain ld.ca (C2 and C4)
set -x
for r in 1 2; do
for v in relaxed ldca; do
cp build/variants/liblobster_$v.so paper_2503_21937_b200/liblobster.so
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --serial > gpurun_out/ab_$v.json 2>/dev/null
python - <<PY
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1])
print('$v C2', round(d['ms_per_step'],2), 'frac', round(d['roofline']['frac'],4), 'us/launch', round(d['roofline']['avg_launch_us'],1))
PY
timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab4_$v.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/ab4_$v.json').read().strip().splitlines()[-1]); print('$v C4', round(d['ms_per_step'],3))"
done
done
cp build/variants/liblobster_relaxed.so paper_2503_21937_b200/liblobster.so
