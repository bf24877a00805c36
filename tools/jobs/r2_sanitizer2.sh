#!/bin/bash
# compute-sanitizer over the decode-path additions: route fused into the gate,
# early-started down GEMM (readiness counters), plan-kernel resets
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/san2
CS=/usr/local/cuda/bin/compute-sanitizer
K="route_in_gate or early_down"
timeout 1200 $CS --tool memcheck python -m pytest tests/test_gpu_layer.py -m gpu -q -p no:cacheprovider -k "$K" > gpurun_out/san2/memcheck.log 2>&1; tail -2 gpurun_out/san2/memcheck.log
timeout 1200 $CS --tool racecheck --racecheck-report hazard --kernel-name-exclude kns=grouped_gemm_kernel python -m pytest tests/test_gpu_layer.py -m gpu -q -p no:cacheprovider -k "$K" > gpurun_out/san2/racecheck.log 2>&1; tail -2 gpurun_out/san2/racecheck.log
timeout 1200 $CS --tool synccheck python -m pytest tests/test_gpu_layer.py -m gpu -q -p no:cacheprovider -k "$K" > gpurun_out/san2/synccheck.log 2>&1; tail -2 gpurun_out/san2/synccheck.log
