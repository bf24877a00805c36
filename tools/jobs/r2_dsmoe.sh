# DS-MoE like-for-like: baseline tests + bench (round 2)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_baseline.py tests/test_gpu_layer.py tests/test_gpu_multiprocess.py -q -rf -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
tail -25 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -5 gpurun_out/bench.err
