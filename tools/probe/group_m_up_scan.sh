#!/bin/bash
# Up-GEMM rasterisation scan (SMOE_GROUP_M_UP: m-blocks per group; < 0: n-blocks per group).
out=gpurun_out/group_m_up_scan.jsonl
: > $out
for rep in 1 2; do
  for cfg in mixtral qwen2_57b; do
    for g in 0 8 16 4 -4 -16; do
      SMOE_GROUP_M_UP=$g timeout 300 python tools/latency.py --config $cfg --tokens 16384 --reps 20 >> $out 2>>gpurun_out/group_m_up_scan.err
    done
  done
done
