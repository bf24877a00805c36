#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/cgfull
for cg in 1 2; do
  timeout 600 ncu --set full --clock-control none -k regex:grouped_gemm -s 2 -c 1 -f -o gpurun_out/cgfull/up_$cg python tools/probe/cg_up_ncu.py $cg > /dev/null 2>&1
  ncu -i gpurun_out/cgfull/up_$cg.ncu-rep --page raw --csv > gpurun_out/cgfull/raw_$cg.csv 2>/dev/null
  rm -f gpurun_out/cgfull/up_$cg.ncu-rep
done
ls -la gpurun_out/cgfull
