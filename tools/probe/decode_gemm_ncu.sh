#!/bin/bash
# ncu --set full of the two expert GEMMs in a warm 64-token forward (no cache
# flush): why DSV2-Lite's up GEMM streams w13 at ~0.7 of HBM peak while
# Mixtral's reaches ~0.9.
mkdir -p gpurun_out
for cfg in dsv2_lite mixtral; do
  timeout 600 ncu --set full --clock-control none --cache-control none --import-source on \
    -k "regex:grouped_gemm" -s 4 -c 2 -f -o gpurun_out/dec_gemm_$cfg \
    python tools/latency.py --config $cfg --tokens 64 --reps 1 > gpurun_out/dec_gemm_$cfg.log 2>&1
  ncu -i gpurun_out/dec_gemm_$cfg.ncu-rep --page raw --csv > gpurun_out/dec_gemm_${cfg}_raw.csv 2>/dev/null
  ncu -i gpurun_out/dec_gemm_$cfg.ncu-rep --page details --csv > gpurun_out/dec_gemm_${cfg}_details.csv 2>/dev/null
done
python tools/latency.py --config dsv2_lite --tokens 64,128 --reps 50 > gpurun_out/dec_lat_dsv2.jsonl 2>&1
ls -la gpurun_out | tail
