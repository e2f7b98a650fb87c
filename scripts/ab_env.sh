# A/B env switches on one build: bash scripts/ab_env.sh CONFIG "ENV1=.. ENV2=.." reps
set +x
mkdir -p gpurun_out
C=${1:-C2}; ENVS=${2:-"X=0"}; REPS=${3:-2}
for rep in $(seq $REPS); do for e in $ENVS; do
env $e timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; print('$C', '$e', 'ms %.2f'%d['ms_per_step'], 'rf_us %s'%(round(r['avg_launch_us'],1) if 'avg_launch_us' in r else '-'), 'frac %.3f'%r['frac'], {k:round(v,2) for k,v in d['phases_ms'].items()})"
done; done
