#!/bin/bash
# ncu evidence for a round (run under gpurun; outputs in gpurun_out/):
#   launch list of the bench command, and --set full captures of the two hot
#   kernels at p = 26 (the eager first cycle's 26th launch of each).
set -u
R=${1:-r2}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 400 --csv --log-file gpurun_out/${R}_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${R}_bench_under_ncu.txt 2>&1
for K in lagged_update_kernel mdot_spmv7; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 25 -c 1 \
      -o gpurun_out/${R}_prof_$K -f python bench.py --steps 1 --warmup 3 --no-cpu \
      > gpurun_out/${R}_prof_$K.log 2>&1
done
