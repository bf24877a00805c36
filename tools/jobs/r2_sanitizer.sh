#!/bin/bash
# compute-sanitizer over the round-2 kernels (split N'=64 gate epilogue, wide gate,
# DS-MoE pipeline stages, ceo scoring, toy chain) + the new -inf mask cases
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/sanitizer
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 python -m pytest tests/test_gpu_gate_semantics.py -m gpu -q -p no:cacheprovider -k "minus_inf" > gpurun_out/sanitizer/masks_plain.log 2>&1; echo masks rc=$?; tail -2 gpurun_out/sanitizer/masks_plain.log
timeout 1200 $CS --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_gate_semantics.py -m gpu -q -p no:cacheprovider -k "ties and 64" > gpurun_out/sanitizer/racecheck_gate64.log 2>&1; echo race rc=$?; tail -3 gpurun_out/sanitizer/racecheck_gate64.log
timeout 1200 $CS --tool synccheck python -m pytest tests/test_gpu_gate_semantics.py -m gpu -q -p no:cacheprovider -k "ties and 64" > gpurun_out/sanitizer/synccheck_gate64.log 2>&1; echo sync rc=$?; tail -3 gpurun_out/sanitizer/synccheck_gate64.log
timeout 1200 $CS --tool memcheck python -m pytest tests/test_gpu_gate_semantics.py -m gpu -q -p no:cacheprovider -k "ties or (minus_inf and 64)" > gpurun_out/sanitizer/memcheck_gate.log 2>&1; echo mem rc=$?; tail -3 gpurun_out/sanitizer/memcheck_gate.log
timeout 1200 $CS --tool memcheck python -m pytest tests/test_gpu_baseline.py tests/test_gpu_solver.py tests/test_gpu_toy_chain.py -m gpu -q -p no:cacheprovider -k "not multiprocess and not distributed" > gpurun_out/sanitizer/memcheck_pipeline.log 2>&1; echo mem2 rc=$?; tail -3 gpurun_out/sanitizer/memcheck_pipeline.log
