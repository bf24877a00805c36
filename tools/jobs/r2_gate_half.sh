#!/bin/bash
# 64-row gate tiles (two CTAs per SM): parity with HALF forced on, then cold-L2 gate times
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/half
SMOE_GATE_HALF=1 timeout 900 python -m pytest tests/test_gpu_gate_semantics.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider > gpurun_out/half/tests_half1.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/half/tests_half1.log
for rep in 1 2; do
for H in 0 1; do
  SMOE_GATE_HALF=$H SMOE_PROBE_CFGS=mixtral,dsv2_lite,qwen2_57b,deepseek_v2 timeout 600 python tools/stage_probe.py --stages gate --flush >> gpurun_out/half/probe.jsonl 2>>gpurun_out/half/probe.err
  SMOE_GATE_HALF=$H SMOE_PROBE_CFGS=mixtral,dsv2_lite,qwen2_57b timeout 600 python tools/stage_probe.py --stages gate --flush --tokens 64 >> gpurun_out/half/probe.jsonl 2>>gpurun_out/half/probe.err
  SMOE_GATE_HALF=$H SMOE_PROBE_CFGS=mixtral,dsv2_lite timeout 600 python tools/stage_probe.py --stages gate --flush --tokens 4096 >> gpurun_out/half/probe.jsonl 2>>gpurun_out/half/probe.err
done
done
cut -c1-160 gpurun_out/half/probe.jsonl; tail -3 gpurun_out/half/probe.err
for H in 0 1; do
  SMOE_GATE_HALF=$H timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gate_tc -c 3 --csv --log-file gpurun_out/half/ncu_$H.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dsmoe --no-decode > /dev/null 2>&1
done
grep -h "gpu__time\|dram_throughput" gpurun_out/half/ncu_*.csv | cut -c1-20,200-400
