#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/gtl
export SMOE_LIB=$PWD/paper_2503_04398_b200/libsmoe_gateprobe.so
for cn in "dsv2_lite 16384" "dsv2_lite 64" "mixtral 16384" "qwen2_57b 16384" "mixtral 64"; do
  set -- $cn
  for H in 0 1; do
    SMOE_GATE_HALF=$H timeout 300 python tools/probe/gate_timeline.py $1 $2 | sed "s/}\$/, \"half\": $H}/" >> gpurun_out/gtl/timeline.jsonl 2>> gpurun_out/gtl/err.txt
  done
done
cat gpurun_out/gtl/timeline.jsonl; tail -3 gpurun_out/gtl/err.txt
