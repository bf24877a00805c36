#!/bin/bash
# wave-synchronised producers of the down GEMM (SMOE_GEMM_SYNC_EVERY): DRAM
# bytes / clock / tensor pipe (ncu, single pass) and bench stage times
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/sync
B="bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dsmoe --no-decode"
SMOE_GEMM_SYNC_EVERY=16 timeout 600 python -m pytest tests/test_gpu_layer.py -m gpu -q -x -p no:cacheprovider > gpurun_out/sync/tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/sync/tests.log
for cfg in mixtral qwen2_57b; do
  for S in 0 8 16 32 64; do
    SMOE_GEMM_SYNC_EVERY=$S timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k "regex:grouped_gemm_kernel" -c 4 --csv --log-file gpurun_out/sync/ncu_${cfg}_$S.csv \
      python $B --config $cfg > /dev/null 2>&1
  done
done
for rep in 1 2 3; do
  for cfg in mixtral qwen2_57b; do
    for S in 0 16 32; do
      SMOE_GEMM_SYNC_EVERY=$S timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-dsmoe --no-decode --config $cfg \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':'$cfg','S':$S,'rep':$rep,'value':d['value'],'ms':d['ms_per_step'],'down_ms':d['stages_ms']['expert_down'],'up_ms':d['stages_ms']['expert_up'],'mhz':d['clocks']['sm_mhz']}))" >> gpurun_out/sync/bench_ab.jsonl
    done
  done
done
cat gpurun_out/sync/bench_ab.jsonl
