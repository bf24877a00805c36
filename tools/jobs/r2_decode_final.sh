#!/bin/bash
# per-kernel device times of one steady-state 64-token forward (the layer has
# just run a 2 048-token batch), final round-2 code, warm L2 (no flush)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/decfinal
for cfg in dsv2_lite mixtral qwen2_57b; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/decfinal/decode_kernels_$cfg.csv python tools/probe/decode_steady.py $cfg 1 > /dev/null 2>&1
  python tools/ncu_csv.py gpurun_out/decfinal/decode_kernels_$cfg.csv | tail -12
done
