#!/bin/bash
# usage: tools/ncu_metrics.sh <out-name> <kernel-regex> <skip> <count> [metrics]
# Writes gpurun_out/<out-name>.csv (ncu --csv) for the bench command.
mkdir -p gpurun_out
M=${5:-gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum}
timeout 300 ncu --metrics "$M" --clock-control none -k "regex:$2" -s "$3" -c "$4" --csv \
  --log-file "gpurun_out/$1.csv" python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dsmoe \
  > /dev/null 2>&1
echo "wrote gpurun_out/$1.csv"
