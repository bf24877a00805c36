#!/bin/bash
# Per-kernel device time of a warm 64-token forward (ncu, no cache flush, no clock lock):
# the last forward of latency.py's eager loop.
for cfg in dsv2_lite mixtral; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
    -k "regex:plan_|srs_|gate_tc|route_|dispatch|grouped_gemm|combine_sag" --csv --log-file gpurun_out/decode_kernels_$cfg.csv \
    python tools/latency.py --config $cfg --tokens 64 --reps 3 > /dev/null 2>&1
done
