#!/bin/bash
# down GEMM: SM pair (256-row tiles) vs one SM (128-row tiles) by rows per expert
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/pair
for rep in 1 2; do
for cfg in deepseek_v2 dsv2_lite qwen2_57b; do
  for R in 64 1024; do
    SMOE_GEMM_PAIR_MIN_ROWS=$R timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu --no-dsmoe --no-decode \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':'$cfg','R':$R,'rep':$rep,'value':d['value'],'down_ms':d['stages_ms']['expert_down'],'up_ms':d['stages_ms']['expert_up'],'mhz':d['clocks']['sm_mhz']}))" >> gpurun_out/pair/ab.jsonl
  done
done
done
cat gpurun_out/pair/ab.jsonl
