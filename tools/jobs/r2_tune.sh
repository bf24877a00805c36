#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/tune
timeout 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_gemm.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider > gpurun_out/tune/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/tune/tests.log
for i in 1 2; do
  for cfg in mixtral qwen2_57b dsv2_lite; do
    timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu --no-dsmoe --no-decode > gpurun_out/tune/b_${cfg}_$i.json 2>gpurun_out/tune/b_${cfg}_$i.err
    timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu --no-dsmoe --no-decode --no-tune > gpurun_out/tune/n_${cfg}_$i.json 2>gpurun_out/tune/n_${cfg}_$i.err
    python -c "
import json
a=json.load(open('gpurun_out/tune/b_${cfg}_$i.json')); b=json.load(open('gpurun_out/tune/n_${cfg}_$i.json'))
print('$cfg', 'tuned', round(a['value']/1e6,3), a['up_gemm_schedule'], a['clocks']['sm_mhz'], '| untuned', round(b['value']/1e6,3), b['clocks']['sm_mhz'])"
  done
done
