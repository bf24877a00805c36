#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/cgup
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for cfg in mixtral qwen2_57b; do
for cg in 1 2 1 2; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:grouped_gemm -c 8 --csv --log-file gpurun_out/cgup/${cfg}_$cg.csv python tools/probe/cg_up_ncu.py $cg $cfg > /dev/null 2>&1
  python - "$cfg" "$cg" <<'PY'
import csv,sys,collections
d=collections.OrderedDict()
for r in csv.reader(open(f'gpurun_out/cgup/{sys.argv[1]}_{sys.argv[2]}.csv')):
    if len(r)<10 or r[0]=='ID': continue
    if 'grouped_gemm_kernel<1,' not in r[4]: continue
    d.setdefault(r[0],{})[r[-3]]=float(r[-1].replace(',',''))
v=list(d.values())[-2:]
for x in v:
    print(sys.argv[1], 'cg', sys.argv[2], round(x['dram__bytes_read.sum']/1e9,2),'GB', round(x['gpu__time_duration.sum']/1e3,1),'us', round(x['sm__cycles_elapsed.avg.per_second']/1e9,3),'GHz', x['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'],'%')
PY
done
done
