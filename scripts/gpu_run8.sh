# one big-round fused join (max-mult: the second engine) under ncu --set full
LOBSTER_JOIN_TIMING_EVERY=1000000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_rows_direct_k -s 200 -c 2 -o gpurun_out/prof_fj python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --serial > gpurun_out/prof_fj.log 2>&1
tail -3 gpurun_out/prof_fj.log
