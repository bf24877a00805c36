#!/bin/bash
# Gate ring depth at decode and full size: 2x4 (default) vs deep 1x(9-12).
out=gpurun_out/gate_ring_deep.jsonl
: > $out
for rep in 1 2; do
  for ring in 2 0; do
    for t in 64 512 16384; do
      SMOE_GATE_RING=$ring timeout 300 python tools/stage_probe.py --stages gate --tokens $t >> $out 2>>gpurun_out/gate_ring_deep.err
    done
    SMOE_GATE_RING=$ring timeout 300 python tools/latency.py --config dsv2_lite --tokens 64,16384 --reps 40 >> $out 2>>gpurun_out/gate_ring_deep.err
  done
done
