#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_narrow5.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_narrow5.log
for cfg in dsv2_lite mixtral qwen2_57b; do
  for nr in 0 16 0 16; do
    SMOE_GEMM_NARROW_MAX_ROWS=$nr timeout 300 python tools/latency.py --config $cfg --tokens 64,128 --reps 50 \
      >> gpurun_out/narrow5_ab.jsonl 2>> gpurun_out/narrow5_ab.err
  done
done
tail -3 gpurun_out/gpu_tests_narrow5.log
