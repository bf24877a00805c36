# bench lines of every model config (round 2)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for cfg in dsv2_lite qwen2_57b deepseek_v2; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "$cfg rc=$?"
done
timeout 300 python tools/stage_probe.py --stages gate --tokens 16384 > gpurun_out/gate_probe_16k.jsonl 2>&1
SMOE_PROBE_CFGS=deepseek_v2 timeout 300 python tools/stage_probe.py --stages gate,srs > gpurun_out/gate_probe_dsv2.jsonl 2>&1
cat gpurun_out/gate_probe_dsv2.jsonl | cut -c1-150
