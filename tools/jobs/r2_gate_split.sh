#!/bin/bash
# N' = 64 gate with two epilogue threads per row (default) vs one (variant nosplit)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/gsplit
timeout 900 python -m pytest tests/test_gpu_gate_semantics.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py tests/test_gpu_toy_chain.py tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gsplit/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gsplit/tests.log
for lib in gateprobe gateprobe_nosplit; do
  for cn in "dsv2_lite 16384" "dsv2_lite 64" "qwen2_57b 16384" "qwen2_57b 64"; do
    set -- $cn
    SMOE_LIB=$PWD/paper_2503_04398_b200/libsmoe_$lib.so timeout 300 python tools/probe/gate_timeline.py $1 $2 | tail -1 | sed "s/}\$/, \"lib\": \"$lib\"}/" >> gpurun_out/gsplit/timeline.jsonl 2>> gpurun_out/gsplit/err.txt
  done
done
cut -c1-260 gpurun_out/gsplit/timeline.jsonl
for rep in 1 2; do
for lib in libsmoe.so libsmoe_nosplit.so; do
  for cfg in dsv2_lite qwen2_57b; do
    SMOE_LIB=$PWD/paper_2503_04398_b200/$lib timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu --no-dsmoe \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$lib','cfg':'$cfg','value':d['value'],'gate_us':d['stages_ms']['gate']*1e3,'decode_us':d['decode']['us_per_step']}))" >> gpurun_out/gsplit/bench.jsonl
  done
done
done
cat gpurun_out/gsplit/bench.jsonl
