# decode movers: GPU suite + latency + per-kernel launch list (round 2)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
tail -8 gpurun_out/gpu_tests.log
for cfg in dsv2_lite mixtral qwen2_57b; do timeout 300 python tools/latency.py --config $cfg --tokens 64,256 ; done > gpurun_out/latency.jsonl 2>gpurun_out/latency.err
cat gpurun_out/latency.jsonl | cut -c1-160
for cfg in dsv2_lite mixtral; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
    -k "regex:plan_|srs_|gate_tc|route_|dispatch|grouped_gemm|combine_sag" --csv --log-file gpurun_out/decode_kernels_$cfg.csv \
    python tools/latency.py --config $cfg --tokens 64 --reps 3 > /dev/null 2>&1
done
python tools/ncu_csv.py gpurun_out/decode_kernels_dsv2_lite.csv | tail -9
