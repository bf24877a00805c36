cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_solver.py tests/test_gpu_golden.py -q -rf -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/gpu_tests.log
timeout 300 python tools/ceo_bench.py > gpurun_out/ceo_bench.json 2>&1; cat gpurun_out/ceo_bench.json
timeout 300 python tools/ceo_bench.py --tokens 102400 --experts 64 --clusters 8 >> gpurun_out/ceo_bench.json 2>&1; tail -1 gpurun_out/ceo_bench.json
if [ -d .refcopy ]; then (cd .refcopy && timeout 600 python ../tools/ref_suite/shim.py pkg pkg/tests -q -p no:cacheprovider -rA > ../gpurun_out/ref_suite.log 2>&1; echo rc=$? >> ../gpurun_out/ref_suite.log); tail -3 gpurun_out/ref_suite.log; fi
