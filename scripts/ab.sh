# A/B two builds on the same box: bash scripts/ab.sh "head new" "C2 C3 C4" [reps]
set +x
mkdir -p gpurun_out
LIBS=${1:-head new}; CFGS=${2:-C2}; REPS=${3:-2}
for rep in $(seq $REPS); do for c in $CFGS; do for lib in $LIBS; do
cp ab/$lib.so paper_2503_21937_b200/liblobster.so
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; print('$c', '$lib', 'ms %.2f'%d['ms_per_step'], 'rf_us %s'%(round(r['avg_launch_us'],1) if 'avg_launch_us' in r else '-'), 'frac %.3f'%r['frac'], {k:round(v,2) for k,v in d['phases_ms'].items()})"
done; done; done
