#!/bin/bash
# why the synced down GEMM idles: ncu --set full of it (Qwen2 16K) with and
# without wave sync, and the sync with row-major (untiled) weights
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/sync3
B="bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dsmoe --no-decode --config qwen2_57b"
for v in "0 0" "32 0" "32 1"; do
  set -- $v
  SMOE_GEMM_SYNC_EVERY=$1 SMOE_UNTILED_WEIGHTS=$2 timeout 600 ncu --set full --clock-control none -k "regex:grouped_gemm" -s 2 -c 2 -f \
    -o gpurun_out/sync3/full_$1_$2 python $B > gpurun_out/sync3/log_$1_$2.txt 2>&1
  ncu -i gpurun_out/sync3/full_$1_$2.ncu-rep --page raw --csv > gpurun_out/sync3/raw_$1_$2.csv 2>/dev/null
  ncu -i gpurun_out/sync3/full_$1_$2.ncu-rep --page details --csv > gpurun_out/sync3/details_$1_$2.csv 2>/dev/null
  rm -f gpurun_out/sync3/full_$1_$2.ncu-rep
done
ls -la gpurun_out/sync3
