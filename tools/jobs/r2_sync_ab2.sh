#!/bin/bash
# wave sync with run-ahead slack: (S, lag) grid, ncu DRAM / clock / tensor pipe of the down GEMM
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/sync2
B="bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dsmoe --no-decode"
for cfg in mixtral qwen2_57b; do
  for SL in 0:1 16:1 16:2 16:4 32:1 32:2 8:2 8:4 64:1; do
    S=${SL%:*}; L=${SL#*:}
    SMOE_GEMM_SYNC_EVERY=$S SMOE_GEMM_SYNC_LAG=$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k "regex:grouped_gemm" -c 4 --csv --log-file gpurun_out/sync2/ncu_${cfg}_${S}_${L}.csv \
      python $B --config $cfg > /dev/null 2>&1
  done
done
python - <<'PY'
import csv,glob,collections
for f in sorted(glob.glob('gpurun_out/sync2/ncu_*.csv')):
    d=collections.OrderedDict()
    for r in csv.reader(open(f)):
        if len(r)<10 or r[0]=='ID': continue
        if '<2, 2' not in r[4]: continue
        d.setdefault(r[0],{})[r[-3]]=float(r[-1].replace(',',''))
    for k,v in d.items():
        print(f.split('/')[-1], round(v['dram__bytes_read.sum']/1e9,2),'GB', round(v['gpu__time_duration.sum']/1e3,1),'us', round(v['sm__cycles_elapsed.avg.per_second']/1e9,3),'GHz', v['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'],'%')
PY
