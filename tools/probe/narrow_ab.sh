#!/bin/bash
# Narrow GEMM m-blocks (32 rows, 5-stage weight ring) vs 128-row tiles at
# decode-sized batches: layer latency (eager + graph) and output identity.
mkdir -p gpurun_out
for cfg in dsv2_lite mixtral qwen2_57b; do
  for nr in 0 16 0 16; do
    SMOE_GEMM_NARROW_MAX_ROWS=$nr timeout 300 python tools/latency.py --config $cfg --tokens 64,128,256 --reps 50 \
      >> gpurun_out/narrow_ab.jsonl 2>> gpurun_out/narrow_ab.err
  done
done
python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/narrow_tests.log 2>&1; echo rc=$? >> gpurun_out/narrow_tests.log
for cfg in dsv2_lite mixtral; do
  SMOE_GEMM_NARROW_MAX_ROWS=16 timeout 600 ncu --set full --clock-control none --cache-control none \
    -k "regex:grouped_gemm" -s 4 -c 2 -f -o gpurun_out/dec_gemm_narrow_$cfg \
    python tools/latency.py --config $cfg --tokens 64 --reps 1 > /dev/null 2>&1
  ncu -i gpurun_out/dec_gemm_narrow_$cfg.ncu-rep --page raw --csv > gpurun_out/dec_gemm_narrow_${cfg}_raw.csv 2>/dev/null
done
tail -3 gpurun_out/narrow_tests.log
