# DRAM bytes + duration of every launch of the dominant kernel (metrics-only pass over one C2 run)
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:${1:-join_rows_direct} --csv --log-file gpurun_out/traffic.csv python scripts/profile_c2.py 3,1 > /dev/null 2>&1
wc -l gpurun_out/traffic.csv
