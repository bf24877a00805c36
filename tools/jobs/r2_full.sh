set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -rf > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
(cd .refcopy && timeout 600 python ../tools/ref_suite/shim.py pkg pkg/tests -q -p no:cacheprovider -rA > ../gpurun_out/ref_suite.log 2>&1; echo rc=$? >> ../gpurun_out/ref_suite.log)
tail -3 gpurun_out/ref_suite.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 600 gpurun_out/bench.json
