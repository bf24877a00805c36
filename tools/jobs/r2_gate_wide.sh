#!/bin/bash
# N' = 48/64 gates through the shared-memory tournament epilogue (default build)
# vs the register max-tree epilogue (variant reg64): parity, timeline, stage times
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/gwide
timeout 900 python -m pytest tests/test_gpu_gate_semantics.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py tests/test_gpu_toy_chain.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gwide/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gwide/tests.log
for lib in gateprobe gateprobe64; do
  for cn in "dsv2_lite 16384" "dsv2_lite 64" "qwen2_57b 16384" "qwen2_57b 64"; do
    set -- $cn
    SMOE_LIB=$PWD/paper_2503_04398_b200/libsmoe_$lib.so timeout 300 python tools/probe/gate_timeline.py $1 $2 | tail -1 | sed "s/}\$/, \"lib\": \"$lib\"}/" >> gpurun_out/gwide/timeline.jsonl 2>> gpurun_out/gwide/err.txt
  done
done
cut -c1-260 gpurun_out/gwide/timeline.jsonl
for rep in 1 2; do
for lib in libsmoe.so libsmoe_reg64.so; do
  for cfg in dsv2_lite qwen2_57b; do
    SMOE_LIB=$PWD/paper_2503_04398_b200/$lib timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu --no-dsmoe \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$lib','cfg':'$cfg','value':d['value'],'gate_us':d['stages_ms']['gate']*1e3,'decode_us':d['decode']['us_per_step']}))" >> gpurun_out/gwide/bench.jsonl
  done
done
done
cat gpurun_out/gwide/bench.jsonl
