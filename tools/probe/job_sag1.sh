python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_sag1.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_sag1.log
tail -3 gpurun_out/gpu_tests_sag1.log
for i in 1 2; do python bench.py --no-cpu --steps 30 > gpurun_out/bench_sag1_$i.json; done
