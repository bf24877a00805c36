#!/bin/bash
# Scan the down-GEMM rasterisation group size under ncu (DRAM bytes, tensor %, time).
for gm in 1 2 3 5 8 16; do
  SMOE_GROUP_M_DOWN=$gm timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"grouped_gemm_kernel<2, 2>" -s 1 -c 2 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dsmoe 2>/dev/null | grep grouped_gemm | awk -v gm=$gm -F'","' '{print "gm=" gm, $(NF-2), $NF}'
done
