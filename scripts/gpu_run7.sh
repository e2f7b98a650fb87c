for pf in 1 0 1 0; do
LOBSTER_FJ_PREFETCH=$pf timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --serial > gpurun_out/b_pf$pf.json 2>&1
python - <<PY
import json; d=json.loads(open('gpurun_out/b_pf$pf.json').read().strip().splitlines()[-1])
print('prefetch=$pf', round(d['ms_per_step'],2), 'frac', round(d['roofline']['frac'],4), 'us/launch', round(d['roofline']['avg_launch_us'],1))
PY
done
