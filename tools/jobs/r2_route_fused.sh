#!/bin/bash
# route fused into the gate (n <= 128): parity suites + ABBA decode A/B
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/rfuse
timeout 1500 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fuzz.py tests/test_gpu_gate_semantics.py tests/test_gpu_multiprocess.py tests/test_gpu_toy_chain.py tests/test_gpu_baseline.py -m gpu -q -x -p no:cacheprovider > gpurun_out/rfuse/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/rfuse/tests.log
for cfg in dsv2_lite mixtral qwen2_57b; do
  timeout 600 python tools/decode_ab.py --config $cfg --tokens 64 --opt 9=1,0 --rounds 8 >> gpurun_out/rfuse/ab.jsonl 2>> gpurun_out/rfuse/err.txt
done
python - <<'PY'
import json
by={}
for l in open('gpurun_out/rfuse/ab.jsonl'):
    d=json.loads(l); by.setdefault(d['config'],{})[d['value']]=(d['rounds_us'], d['identical_to_first'])
for c,v in by.items():
    on,off=v[1][0],v[0][0]
    diffs=sorted(b-a for a,b in zip(on,off))
    print(c, 'identical', v[0][1], 'per-round off-on median', round(diffs[len(diffs)//2],2), [round(x,1) for x in diffs])
PY
