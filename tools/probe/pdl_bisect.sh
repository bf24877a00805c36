#!/bin/bash
# Which layer stage's early launch (SMOE_PDL_STAGES bit mask, bit = stage id)
# changes the 16K-token step time.
out=gpurun_out/pdl_bisect.jsonl
: > $out
for rep in 1 2; do
  for cfg in mixtral qwen2_57b; do
    for m in 0x00 0xff 0x1f 0x20 0x40 0x80 0x60; do
      SMOE_PDL_STAGES=$m timeout 300 python tools/latency.py --config $cfg --tokens 16384 --reps 20 >> $out 2>>gpurun_out/pdl_bisect.err
    done
  done
done
