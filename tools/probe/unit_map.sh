#!/bin/bash
# Up-GEMM CTA -> tile mapping: blockIdx (0) vs %smid-derived (1: smid, 2: even
# SMs first, 3: halves interleaved), plain launch.  Plus the blockIdx -> smid map.
out=gpurun_out/unit_map.jsonl
: > $out
./tools/probe/smid_map > gpurun_out/smid_map.jsonl 2>&1
for rep in 1 2; do
  for cfg in mixtral qwen2_57b; do
    for um in 0 1 2 3; do
      SMOE_GEMM_UNIT_MAP=$um SMOE_PDL_STAGES=0xdf timeout 300 python tools/latency.py --config $cfg --tokens 16384 --reps 20 >> $out 2>>gpurun_out/unit_map.err
    done
  done
done
