#!/bin/bash
# up GEMM on SM pairs: smaller A-resident groups (group_m 8 / 4 / 2 m-blocks of 256 rows)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/cg2gm
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct"
for cfg in mixtral qwen2_57b; do
for v in "1 0" "2 0" "2 8" "2 4" "2 2" "2 -2"; do
  set -- $v
  SMOE_GROUP_M_UP=$2 timeout 300 ncu --metrics $M --clock-control none -k regex:grouped_gemm -c 8 --csv --log-file gpurun_out/cg2gm/${cfg}_$1_$2.csv python tools/probe/cg_up_ncu.py $1 $cfg > /dev/null 2>&1
  python - "$cfg" "$1" "$2" <<'PY'
import csv,sys,collections
d=collections.OrderedDict()
for r in csv.reader(open(f'gpurun_out/cg2gm/{sys.argv[1]}_{sys.argv[2]}_{sys.argv[3]}.csv')):
    if len(r)<10 or r[0]=='ID' or 'grouped_gemm_kernel<1,' not in r[4]: continue
    d.setdefault(r[0],{})[r[-3]]=float(r[-1].replace(',',''))
for x in list(d.values())[-2:]:
    print(sys.argv[1], 'cg', sys.argv[2], 'gm', sys.argv[3], round(x['dram__bytes_read.sum']/1e9,2),'GB', round(x['gpu__time_duration.sum']/1e3,1),'us', round(x['sm__cycles_elapsed.avg.per_second']/1e9,3),'GHz', round(x['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'],1),'%', 'L2hit', round(x['lts__t_sector_hit_rate.pct'],1))
PY
done
done
