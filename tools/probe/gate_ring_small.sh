out=gpurun_out/gate_ring_small.jsonl; : > $out
for rep in 1 2; do for ring in 1 2 4; do for t in 64 512; do
  SMOE_GATE_RING=$ring timeout 300 python tools/stage_probe.py --stages gate --tokens $t >> $out
done; done; done
