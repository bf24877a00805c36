#!/bin/bash
# why the in-layer down GEMM moves 8 GB of DRAM while the same shape standalone moves 5.1 GB
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/downdiag
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
B="bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dsmoe --no-decode"
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics $M --clock-control none -k regex:grouped_gemm -c 4 --csv --log-file gpurun_out/downdiag/$tag.csv python $B > /dev/null 2>&1; }
run layer_default X=1
run layer_nopdl_down SMOE_PDL_STAGES=159
run layer_untiled SMOE_UNTILED_WEIGHTS=1
run layer_nopdl_all SMOE_PDL=0
SMOE_PROBE_MS=4036,4180,4038,4045,4017,4121,4118,4213 timeout 300 ncu --metrics $M --clock-control none -k regex:grouped_gemm -s 5 -c 2 --csv --log-file gpurun_out/downdiag/standalone_skew.csv python tools/probe/gemm_splitk_probe.py 2 8 4352 14336 4096 > /dev/null 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:grouped_gemm -s 5 -c 2 --csv --log-file gpurun_out/downdiag/standalone_even.csv python tools/probe/gemm_splitk_probe.py 2 8 4096 14336 4096 > /dev/null 2>&1
python - <<'PY'
import csv,glob,collections
for f in sorted(glob.glob('gpurun_out/downdiag/*.csv')):
    d=collections.OrderedDict()
    for r in csv.reader(open(f)):
        if len(r)<10 or r[0]=='ID' or '<2, ' not in r[4]: continue
        d.setdefault(r[0],{})[r[-3]]=float(r[-1].replace(',',''))
    for k,v in d.items():
        print(f.split('/')[-1], round(v['dram__bytes_read.sum']/1e9,2),'GB', round(v['gpu__time_duration.sum']/1e3,1),'us', round(v['sm__cycles_elapsed.avg.per_second']/1e9,3),'GHz', v['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'],'%')
PY
