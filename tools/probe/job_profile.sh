#!/bin/bash
# Round-end evidence: bench line (both arms), per-step launch list, ncu --set full
# of the layer's kernels in the timed step.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err
python bench.py --impl reference > gpurun_out/bench_ref_r1f.json 2> gpurun_out/bench_ref_r1f.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r1f.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
  --no-dsmoe --no-decode > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k "regex:grouped_gemm|gate_tc|srs_kernel|combine_sag|dispatch_kernel" \
  -s 6 -c 6 -f -o gpurun_out/r1f_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu \
  --no-dsmoe --no-decode > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/r1f_full.ncu-rep --page raw --csv > gpurun_out/r1f_full_raw.csv 2>/dev/null
ncu -i gpurun_out/r1f_full.ncu-rep --page details --csv > gpurun_out/r1f_full_details.csv 2>/dev/null
ls -la gpurun_out
for cfg in dsv2_lite qwen2_57b; do
  python bench.py --config $cfg --no-e2e --no-dsmoe > gpurun_out/bench_r1f_$cfg.json 2> gpurun_out/bench_r1f_$cfg.err
done
