#!/bin/bash
# bench lines of the other model configs (all legs but the CPU baseline)
cd "$(dirname "$0")/../.."
TAG=${TAG:-r2}
mkdir -p gpurun_out
for cfg in dsv2_lite qwen2_57b deepseek_v2; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_${TAG}_$cfg.json 2> gpurun_out/bench_${TAG}_$cfg.err; echo "$cfg rc=$?"
done
