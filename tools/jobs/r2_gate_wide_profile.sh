#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/gwp
B="bench.py --config deepseek_v2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-dsmoe --no-decode"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gate_tc -s 1 -c 1 -f -o gpurun_out/gwp/g python $B > gpurun_out/gwp/log.txt 2>&1
ncu -i gpurun_out/gwp/g.ncu-rep --page source --csv --print-source sass > gpurun_out/gwp/source.csv 2>/dev/null
ncu -i gpurun_out/gwp/g.ncu-rep --page raw --csv > gpurun_out/gwp/raw.csv 2>/dev/null
rm -f gpurun_out/gwp/g.ncu-rep
ls -la gpurun_out/gwp
