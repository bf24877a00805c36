#!/bin/bash
# gate ring shape with a cold L2 (ncu, in the bench's step): bytes per row per stage
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/gring
B="bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-dsmoe --no-decode"
for R in 2 1 4 43 2; do
  SMOE_GATE_RING=$R timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gate_tc --csv --log-file gpurun_out/gring/ncu_$R.csv python $B > /dev/null 2>&1
  python - "$R" <<'PY'
import csv,sys,collections
d=collections.defaultdict(dict)
for r in csv.reader(open(f'gpurun_out/gring/ncu_{sys.argv[1]}.csv')):
    if len(r)<10 or r[0]=='ID': continue
    d[r[0]][r[-3]]=float(r[-1].replace(',',''))
ts=[v['gpu__time_duration.sum']/1e3 for v in d.values()]
print(sys.argv[1], [round(t,1) for t in ts], [round(v['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'],1) for v in d.values()])
PY
done
for R in 2 43 2 43; do SMOE_GATE_RING=$R SMOE_PROBE_CFGS=mixtral timeout 300 python tools/stage_probe.py --stages gate --flush | cut -c1-120; done
