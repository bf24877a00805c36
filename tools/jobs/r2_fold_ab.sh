#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/fold
for cfg in dsv2_lite mixtral; do
  timeout 900 python tools/probe/lib_ab.py paper_2503_04398_b200/libsmoe.so paper_2503_04398_b200/libsmoe_nofold.so $cfg 64 4 >> gpurun_out/fold/ab.jsonl 2>> gpurun_out/fold/err.txt
done
cat gpurun_out/fold/ab.jsonl; tail -3 gpurun_out/fold/err.txt
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report hazard --kernel-name kns=gate_tc python -m pytest tests/test_gpu_gate_semantics.py -m gpu -q -p no:cacheprovider -k "ties and 64" > gpurun_out/fold/racecheck_gate_only.log 2>&1; tail -3 gpurun_out/fold/racecheck_gate_only.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report hazard --kernel-name-exclude kns=grouped_gemm python -m pytest tests/test_gpu_gate_semantics.py -m gpu -q -p no:cacheprovider -k "ties and 64" > gpurun_out/fold/racecheck_movers.log 2>&1; tail -3 gpurun_out/fold/racecheck_movers.log
