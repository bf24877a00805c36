#!/bin/bash
# ring shape of the N' = 64 (split-epilogue) gate, cold L2, timeline probe build
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/gring64
export SMOE_LIB=$PWD/paper_2503_04398_b200/libsmoe_gateprobe.so
for r in 1 2; do
for R in 2 1 4; do
  for cn in "dsv2_lite 16384" "dsv2_lite 64" "qwen2_57b 16384"; do
    set -- $cn
    SMOE_GATE_RING=$R timeout 300 python tools/probe/gate_timeline.py $1 $2 | tail -1 | sed "s/}\$/, \"ring\": $R}/" >> gpurun_out/gring64/t.jsonl 2>> gpurun_out/gring64/err.txt
  done
done
done
python - <<'PY'
import json
for l in open('gpurun_out/gring64/t.jsonl'):
    d=json.loads(l); m=d['median_us']
    print(d['config'], d['tokens'], 'ring', d['ring'], 'first', m[3], 'lastTMA', m[2], 'lastMMA', m[4], 'epi_done', m[6], 'exit', m[7])
PY
