#!/bin/bash
# combine+SAG at 3 CTAs per SM (launch bounds) vs 2 (libsmoe_prev.so): bench stage times.
mkdir -p gpurun_out
for rep in 1 2 3; do
  for lib in libsmoe.so libsmoe_prev.so; do
    for cfg in mixtral dsv2_lite qwen2_57b; do
      SMOE_LIB=$PWD/paper_2503_04398_b200/$lib timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-dsmoe --no-cpu --no-decode \
        | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(json.dumps({'lib':'$lib','config':'$cfg','srs_ms':d['stages_ms']['srs'],'dispatch_ms':d['stages_ms']['dispatch'],'ms_per_step':d['ms_per_step']}))" >> gpurun_out/srs_occ.jsonl 2>>gpurun_out/srs_occ.err
    done
  done
done
python -m pytest tests/test_gpu_layer.py tests/test_gpu_collectives.py -q -x > gpurun_out/srs_occ_tests.log 2>&1; echo rc=$? >> gpurun_out/srs_occ_tests.log
