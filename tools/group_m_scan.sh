#!/bin/bash
# Scan the down-GEMM rasterisation group size under ncu (DRAM bytes, tensor %, time).
mkdir -p gpurun_out
for gm in ${GMS:-1 -4 -8 -16 16}; do
  SMOE_GROUP_M_DOWN=$gm timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:grouped_gemm -c 4 --csv --log-file gpurun_out/gm_$gm.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dsmoe > /dev/null 2>&1
done
ls gpurun_out/gm_*.csv
