#!/bin/bash
# early-started down GEMM at decode sizes: parity suites, then interleaved A/B
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/early
timeout 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_gemm.py tests/test_gpu_fuzz.py tests/test_gpu_multiprocess.py tests/test_gpu_gate_semantics.py -m gpu -q -x -p no:cacheprovider > gpurun_out/early/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/early/tests.log
for cfg in dsv2_lite mixtral qwen2_57b; do
  timeout 600 python tools/decode_ab.py --config $cfg --tokens 64 --opt 8=1,0 --rounds 7 >> gpurun_out/early/ab.jsonl 2>> gpurun_out/early/err.txt
  timeout 600 python tools/decode_ab.py --config $cfg --tokens 256 --opt 8=1,0 --rounds 5 >> gpurun_out/early/ab.jsonl 2>> gpurun_out/early/err.txt
done
cut -c1-200 gpurun_out/early/ab.jsonl; tail -3 gpurun_out/early/err.txt
