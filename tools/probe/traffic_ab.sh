#!/bin/bash
# DRAM bytes of the two expert GEMMs (timed-step launch) under layout / launch knobs.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second
for v in "X=1" "SMOE_PDL=0" "SMOE_UNTILED_WEIGHTS=1" "SMOE_UNTILED_WEIGHTS=1 SMOE_PDL=0"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 400 ncu --metrics "$M" --clock-control none -k "regex:grouped_gemm" -s 2 -c 2 --csv \
    --log-file gpurun_out/traffic_$tag.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu \
    --no-dsmoe --no-decode > /dev/null 2>&1
  echo "== $v"; python tools/ncu_csv.py gpurun_out/traffic_$tag.csv
done
