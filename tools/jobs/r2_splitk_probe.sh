#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/splitk
for K in 14336 7168 4096; do
  for GM in 0 1; do
    SMOE_GROUP_M_DOWN=$GM python tools/probe/gemm_splitk_probe.py 2 8 4096 $K 4096 >> gpurun_out/splitk/time.txt 2>&1
    echo "GM=$GM" >> gpurun_out/splitk/time.txt
    SMOE_GROUP_M_DOWN=$GM timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:grouped_gemm -s 5 -c 2 --csv --log-file gpurun_out/splitk/ncu_${K}_$GM.csv \
      python tools/probe/gemm_splitk_probe.py 2 8 4096 $K 4096 > /dev/null 2>&1
  done
done
cat gpurun_out/splitk/time.txt
python - <<'PY'
import csv,glob,collections
for f in sorted(glob.glob('gpurun_out/splitk/ncu_*.csv')):
    d=collections.OrderedDict()
    for r in csv.reader(open(f)):
        if len(r)<10 or r[0]=='ID': continue
        d.setdefault(r[0],{})[r[-3]]=float(r[-1].replace(',',''))
    for k,v in d.items():
        print(f.split('/')[-1], round(v['dram__bytes_read.sum']/1e9,2),'GB', round(v['gpu__time_duration.sum']/1e3,1),'us', round(v['sm__cycles_elapsed.avg.per_second']/1e9,3),'GHz', v['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'],'%')
PY
