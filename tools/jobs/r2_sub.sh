cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest ${PYTEST_FILES:-tests} -m gpu -q -rf -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
tail -30 gpurun_out/gpu_tests.log
