#!/bin/bash
# wave sync x L2 prefetch-ahead of the down GEMM: ncu (DRAM, clock, tensor pipe) + bench stage times
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/sync4
SMOE_GEMM_SYNC_EVERY=32 SMOE_GEMM_PREFETCH_KB=8 timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_gemm.py -m gpu -q -x -p no:cacheprovider > gpurun_out/sync4/tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/sync4/tests.log
B="bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dsmoe --no-decode"
for cfg in qwen2_57b mixtral; do
  for SP in 0:0 0:4 0:8 32:4 32:8 32:16 16:8 64:8; do
    S=${SP%:*}; P=${SP#*:}
    SMOE_GEMM_SYNC_EVERY=$S SMOE_GEMM_PREFETCH_KB=$P timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k "regex:grouped_gemm" -c 4 --csv --log-file gpurun_out/sync4/ncu_${cfg}_${S}_${P}.csv \
      python $B --config $cfg > /dev/null 2>&1
  done
done
python - <<'PY'
import csv,glob,collections
for f in sorted(glob.glob('gpurun_out/sync4/ncu_*.csv')):
    d=collections.OrderedDict()
    for r in csv.reader(open(f)):
        if len(r)<10 or r[0]=='ID': continue
        if '<2, 2' not in r[4]: continue
        d.setdefault(r[0],{})[r[-3]]=float(r[-1].replace(',',''))
    for k,v in d.items():
        print(f.split('/')[-1], round(v['dram__bytes_read.sum']/1e9,2),'GB', round(v['gpu__time_duration.sum']/1e3,1),'us', round(v['sm__cycles_elapsed.avg.per_second']/1e9,3),'GHz', v['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'],'%')
PY
for rep in 1 2; do
  for cfg in mixtral qwen2_57b; do
    for SP in 0:0 32:8 0:8 32:16; do
      S=${SP%:*}; P=${SP#*:}
      SMOE_GEMM_SYNC_EVERY=$S SMOE_GEMM_PREFETCH_KB=$P timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-dsmoe --no-decode --config $cfg \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':'$cfg','S':$S,'P':$P,'rep':$rep,'value':d['value'],'ms':d['ms_per_step'],'down_ms':d['stages_ms']['expert_down'],'up_ms':d['stages_ms']['expert_up'],'mhz':d['clocks']['sm_mhz']}))" >> gpurun_out/sync4/bench_ab.jsonl
    done
  done
done
cat gpurun_out/sync4/bench_ab.jsonl
