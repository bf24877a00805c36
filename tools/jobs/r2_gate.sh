# gate stage probe + GPU suite + bench (round 2)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 300 python tools/stage_probe.py --stages gate,srs > gpurun_out/gate_probe.jsonl 2> gpurun_out/gate_probe.err
timeout 300 python tools/stage_probe.py --stages gate --tokens 64 >> gpurun_out/gate_probe.jsonl 2>>gpurun_out/gate_probe.err
cut -c1-140 gpurun_out/gate_probe.jsonl
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
tail -15 gpurun_out/gpu_tests.log
[ -n "$NO_BENCH" ] || { timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; }
