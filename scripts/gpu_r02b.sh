# Round-2 (session 3) GPU pass: C3 compaction A/B, C1 timeline, tile tests.
# usage: bash scripts/gpu_r02b.sh [what...]
set -x
mkdir -p gpurun_out
for what in "$@"; do
case $what in
tile) timeout 900 python -m pytest tests/test_gpu_tile.py -x -q > gpurun_out/tile.log 2>&1; tail -5 gpurun_out/tile.log ;;
c3ab) for v in 0 1; do
        if [ $v = 1 ]; then export LOBSTER_NO_TILE_COMPACT=1; fi
        timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3_nc$v.json 2> gpurun_out/bench_C3_nc$v.err
        tail -2 gpurun_out/bench_C3_nc$v.err; cut -c1-200 gpurun_out/bench_C3_nc$v.json
      done; unset LOBSTER_NO_TILE_COMPACT ;;
c3nt) for nt in 1024 512; do
        LOBSTER_TILE_THREADS=$nt timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3_nt$nt.json 2> gpurun_out/bench_C3_nt$nt.err
        tail -2 gpurun_out/bench_C3_nt$nt.err; cut -c1-200 gpurun_out/bench_C3_nt$nt.json
      done ;;
c3trace) timeout 300 python scripts/tile_trace_c3.py > gpurun_out/c3trace.txt 2>&1; grep -c sample gpurun_out/c3trace.txt ;;
lookup) timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dmaxmin.py tests/test_gpu_microbatch.py tests/test_gpu_eval.py -x -q > gpurun_out/lookup_tests.log 2>&1; tail -3 gpurun_out/lookup_tests.log
      for v in 1 0; do LOBSTER_LOOKUP_FAST32=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2_lf$v.json 2> gpurun_out/bench_C2_lf$v.err; tail -1 gpurun_out/bench_C2_lf$v.err; cut -c1-200 gpurun_out/bench_C2_lf$v.json; done ;;
c2plog) LOBSTER_LOG=1 timeout 600 python scripts/profile_cfg.py C2P 2 > gpurun_out/c2plog.txt 2>&1; tail -6 gpurun_out/c2plog.txt
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2P.csv python scripts/profile_cfg.py C2P 1 > /dev/null 2>&1
      python scripts/launches.py gpurun_out/launches_C2P.csv 15 ;;
c4) timeout 900 python -m pytest tests/test_gpu_slice.py -x -q > gpurun_out/slice.log 2>&1; tail -2 gpurun_out/slice.log
    timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; tail -1 gpurun_out/bench_C4.err; cut -c1-200 gpurun_out/bench_C4.json
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv python scripts/profile_cfg.py C4 1 > /dev/null 2>&1; python scripts/launches.py gpurun_out/launches_C4.csv 6 ;;
l2w) for v in 1 0 1 0; do LOBSTER_L2_WINDOW=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2_l2w$v.json 2> gpurun_out/bench_C2_l2w$v.err; echo "l2w=$v $(cut -c1-140 gpurun_out/bench_C2_l2w$v.json)"; done
     for v in 1 0; do LOBSTER_L2_WINDOW=$v timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_l2w$v.json 2>/dev/null; echo "C5 l2w=$v $(cut -c1-140 gpurun_out/bench_C5_l2w$v.json)"; done ;;
ex) timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deep.py tests/test_gpu_slice.py tests/test_gpu_microbatch.py -x -q > gpurun_out/ex_tests.log 2>&1; tail -2 gpurun_out/ex_tests.log
    for v in 8 4 16; do LOBSTER_EX_CTAS=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2_ex$v.json 2>/dev/null; echo "ex=$v $(cut -c1-140 gpurun_out/bench_C2_ex$v.json)"; done
    LOBSTER_EX_CTAS=8 timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_ex.json 2>/dev/null; echo "C5 $(cut -c1-140 gpurun_out/bench_C5_ex.json)"
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2e.csv python scripts/profile_c2.py 1,3 > /dev/null 2>&1; python scripts/launches.py gpurun_out/launches_c2e.csv 6 ;;
ex2) for v in 8 64 8 64; do LOBSTER_EX_CTAS=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2_ex$v.json 2>/dev/null; echo "ex=$v $(cut -c1-140 gpurun_out/bench_C2_ex$v.json)"; done
    timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_ex.json 2>/dev/null; echo "C5 $(cut -c1-140 gpurun_out/bench_C5_ex.json)"
    timeout 600 python bench.py --config SG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_SG_ex.json 2>/dev/null; echo "SG $(cut -c1-140 gpurun_out/bench_SG_ex.json)" ;;
cnt) timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slice.py tests/test_gpu_eval.py tests/test_gpu_dmaxmin.py -x -q > gpurun_out/cnt_tests.log 2>&1; tail -2 gpurun_out/cnt_tests.log
    for c in C2 C2 C4 C5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cnt_$c.json 2>/dev/null; echo "$c $(cut -c1-140 gpurun_out/bench_cnt_$c.json)"; done ;;
ex3) timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deep.py tests/test_gpu_microbatch.py tests/test_gpu_dmaxmin.py tests/test_gpu_partition.py -x -q > gpurun_out/ex3_tests.log 2>&1; tail -2 gpurun_out/ex3_tests.log
    for c in C2 C2 C5 SG; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ex3_$c.json 2>/dev/null; echo "$c $(cut -c1-140 gpurun_out/bench_ex3_$c.json)"; done ;;
sort) timeout 2400 python -m pytest tests/ -x -q -m gpu > gpurun_out/sort_tests.log 2>&1; tail -2 gpurun_out/sort_tests.log
    for c in C1 C1 C3 SG C2P; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sort_$c.json 2>/dev/null; echo "$c $(cut -c1-140 gpurun_out/bench_sort_$c.json)"; done ;;
sync1) timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tile.py tests/test_abi.py tests/test_gpu_eval.py -x -q > gpurun_out/sync1_tests.log 2>&1; tail -2 gpurun_out/sync1_tests.log
    for c in C1 C1 C2; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sync1_$c.json 2>/dev/null; echo "$c $(cut -c1-140 gpurun_out/bench_sync1_$c.json)"; done
    LOBSTER_LOG=1 timeout 300 python scripts/profile_cfg.py C1 4 2>&1 | tail -3 ;;
extune) for rep in 1 2; do for cfg in "2 8" "4 8" "2 12" "4 4"; do set -- $cfg; LOBSTER_EX_WPT=$1 LOBSTER_EX_CTAS=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_extune.json 2>/dev/null; echo "wpt=$1 ctas=$2 $(cut -c100-140 gpurun_out/bench_extune.json)"; done; done ;;
skip) timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deep.py tests/test_gpu_dmaxmin.py -x -q > gpurun_out/skip_tests.log 2>&1; tail -2 gpurun_out/skip_tests.log
    for c in C2 C2 C2 C5 SG; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_skip.json 2>/dev/null; echo "$c $(cut -c100-140 gpurun_out/bench_skip.json)"; done ;;
c1log) LOBSTER_LOG=1 timeout 300 python scripts/profile_cfg.py C1 5 > gpurun_out/c1log.txt 2>&1; tail -30 gpurun_out/c1log.txt ;;
c3log) LOBSTER_LOG=1 timeout 300 python scripts/profile_cfg.py C3 3 > gpurun_out/c3log.txt 2>&1; tail -12 gpurun_out/c3log.txt ;;
c3full) timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_fixpoint -s 2 -c 1 -o gpurun_out/prof_tile python scripts/profile_cfg.py C3 2 > gpurun_out/ncu_tile.log 2>&1; tail -2 gpurun_out/ncu_tile.log ;;
configs) for c in C1 C2 C3 C4 C5 C2P SG; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; cut -c1-300 gpurun_out/bench_$c.json; done ;;
esac
done
