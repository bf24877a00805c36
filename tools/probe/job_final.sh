python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_final.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_final.log
tail -3 gpurun_out/gpu_tests_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo rc=$? >> gpurun_out/smoke_final.log; tail -2 gpurun_out/smoke_final.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 600 gpurun_out/bench_final.json
python bench.py --impl reference > gpurun_out/bench_ref_final.json 2>&1
