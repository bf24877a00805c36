#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/race
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool racecheck --racecheck-report hazard --kernel-name-exclude kns=grouped_gemm python -m pytest tests/test_gpu_gate_semantics.py -m gpu -q -p no:cacheprovider -k "ties and 64" > gpurun_out/race/racecheck_all_but_gemm.log 2>&1; tail -2 gpurun_out/race/racecheck_all_but_gemm.log
for cg in 1 2; do
  timeout 600 $CS --tool racecheck --racecheck-report hazard python tools/probe/gemm_splitk_probe.py $cg 2 512 1024 512 > gpurun_out/race/racecheck_gemm_cg$cg.log 2>&1; tail -1 gpurun_out/race/racecheck_gemm_cg$cg.log
done
grep "Error: Potential" gpurun_out/race/racecheck_gemm_cg2.log | head -3
