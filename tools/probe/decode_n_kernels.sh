#!/bin/bash
# Per-kernel device times (warm, no cache flush) of DSV2-Lite forwards at 64 vs 128 tokens.
mkdir -p gpurun_out
for n in 64 128; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --cache-control none \
    -k "regex:plan_|srs_|gate_tc|route_|dispatch|grouped_gemm|combine_sag" --csv --log-file gpurun_out/dsv2_kernels_$n.csv \
    python tools/latency.py --config dsv2_lite --tokens $n --reps 2 > /dev/null 2>&1
done
python tools/probe/../../tools/stage_probe.py --help > /dev/null 2>&1 || true
