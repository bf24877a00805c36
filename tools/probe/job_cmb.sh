python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_cmb.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_cmb.log
tail -3 gpurun_out/gpu_tests_cmb.log
for i in 1 2; do python bench.py --no-cpu --no-dsmoe --no-e2e --steps 30 > gpurun_out/bench_cmb_$i.json; done
for c in dsv2_lite qwen2_57b; do python bench.py --config $c --no-cpu --no-dsmoe --no-e2e --steps 20 > gpurun_out/bench_cmb_$c.json; done
