#!/bin/bash
# plan kernel owns the per-forward resets at decode sizes: layer/golden/multiprocess
# tests + decode latency (graph replay), then the sanitizer pass
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/pfold
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_golden.py tests/test_gpu_multiprocess.py tests/test_gpu_toy_chain.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pfold/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/pfold/tests.log
for cfg in dsv2_lite mixtral qwen2_57b; do
  timeout 300 python tools/latency.py --config $cfg --tokens 64,512 --reps 50 >> gpurun_out/pfold/latency.jsonl 2>> gpurun_out/pfold/latency.err
done
cut -c1-170 gpurun_out/pfold/latency.jsonl
bash tools/jobs/r2_sanitizer.sh
