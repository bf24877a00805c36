#!/bin/bash
# A/B of programmatic dependent launch (SMOE_PDL=0 vs the default stage mask,
# and every stage incl. the up GEMM): eager and CUDA-graph latency, output hashes.
out=${1:-gpurun_out/pdl_ab.jsonl}
: > "$out"
for rep in 1 2; do
  for cfg in mixtral dsv2_lite qwen2_57b; do
    for mode in "SMOE_PDL=0" "SMOE_PDL=1" "SMOE_PDL_STAGES=0xff"; do
      env $mode timeout 300 python tools/latency.py --config $cfg --tokens 64,512,2048,16384 --reps 40 >> "$out" 2>> gpurun_out/pdl_ab.err
    done
  done
done
