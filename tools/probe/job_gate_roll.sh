#!/bin/bash
# Rolled top-k pass loop in the tcgen05 gate epilogue vs the fully unrolled one
# (libsmoe_prev.so): layer latency A/B + gate kernel times (ncu, warm).
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_gate_roll.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_gate_roll.log
bash tools/probe/build_ab.sh paper_2503_04398_b200/libsmoe_prev.so gpurun_out/gate_roll_ab.jsonl 64,512,16384
for lib in libsmoe.so libsmoe_prev.so; do
  for cfg in dsv2_lite mixtral; do
    for n in 64 16384; do
      SMOE_LIB=$PWD/paper_2503_04398_b200/$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
        -k "regex:gate_tc" --csv --log-file gpurun_out/gate_roll_${lib%.so}_${cfg}_$n.csv \
        python tools/latency.py --config $cfg --tokens $n --reps 3 > /dev/null 2>&1
    done
  done
done
tail -2 gpurun_out/gpu_tests_gate_roll.log
