#!/bin/bash
# decode L2 weight prefetch (SMOE_OPT_DECODE_PREFETCH_MB = option 8): interleaved A/B
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for cfg in dsv2_lite mixtral qwen2_57b; do
  timeout 600 python tools/decode_ab.py --config $cfg --tokens 64 --opt 8=0,32,64,96,128 --rounds 7
done > gpurun_out/prefetch_ab.jsonl 2> gpurun_out/prefetch_ab.err
cut -c1-200 gpurun_out/prefetch_ab.jsonl; tail -3 gpurun_out/prefetch_ab.err
