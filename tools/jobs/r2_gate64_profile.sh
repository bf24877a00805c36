#!/bin/bash
# where the N' = 64 gate spends its time (DSV2-Lite 16K): ncu --set full with source
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/gate64
B="bench.py --config dsv2_lite --steps 1 --warmup 1 --no-e2e --no-cpu --no-dsmoe --no-decode"
for H in 0 1; do
  SMOE_GATE_HALF=$H timeout 600 ncu --set full --import-source on --clock-control none -k regex:gate_tc -s 1 -c 1 -f \
    -o gpurun_out/gate64/g_$H python $B > gpurun_out/gate64/log_$H.txt 2>&1
  ncu -i gpurun_out/gate64/g_$H.ncu-rep --page raw --csv > gpurun_out/gate64/raw_$H.csv 2>/dev/null
  ncu -i gpurun_out/gate64/g_$H.ncu-rep --page details --csv > gpurun_out/gate64/details_$H.csv 2>/dev/null
  ncu -i gpurun_out/gate64/g_$H.ncu-rep --page source --csv --print-source sass > gpurun_out/gate64/source_$H.csv 2>/dev/null
done
ls -la gpurun_out/gate64
