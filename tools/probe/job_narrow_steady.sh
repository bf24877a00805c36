#!/bin/bash
# Narrow GEMM on/off in the bench's steady-state decode leg (64 tokens, graph
# replay on a layer that has just run 16 384-token batches).
mkdir -p gpurun_out
for rep in 1 2; do
  for cfg in dsv2_lite mixtral qwen2_57b; do
    for nr in 0 16; do
      SMOE_GEMM_NARROW_MAX_ROWS=$nr timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-dsmoe --no-cpu \
        | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(json.dumps({'config':'$cfg','narrow_max_rows':$nr,'decode_us':d['decode']['us_per_step'],'roofline_us':d['decode']['weight_stream_roofline_us'],'value':d['value']}))" \
        >> gpurun_out/narrow_steady.jsonl 2>> gpurun_out/narrow_steady.err
    done
  done
done
