#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/early2
for cfg in qwen2_57b mixtral dsv2_lite; do
  timeout 600 python tools/decode_ab.py --config $cfg --tokens 64 --opt 8=1,0 --rounds 10 >> gpurun_out/early2/ab.jsonl 2>> gpurun_out/early2/err.txt
done
cut -c1-300 gpurun_out/early2/ab.jsonl
