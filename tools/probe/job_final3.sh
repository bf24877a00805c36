#!/bin/bash
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r1h.json 2> gpurun_out/bench_r1h.err
for cfg in dsv2_lite qwen2_57b; do
  python bench.py --config $cfg > gpurun_out/bench_r1h_$cfg.json 2> gpurun_out/bench_r1h_$cfg.err
done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1h.log 2>&1; echo rc=$? >> gpurun_out/smoke_r1h.log
tail -2 gpurun_out/smoke_r1h.log
