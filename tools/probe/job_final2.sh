#!/bin/bash
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r1g.json 2> gpurun_out/bench_r1g.err
python bench.py --impl reference > gpurun_out/bench_ref_r1g.json 2> gpurun_out/bench_ref_r1g.err
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r1g.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_r1g.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1g.log 2>&1; echo rc=$? >> gpurun_out/smoke_r1g.log
tail -2 gpurun_out/gpu_tests_r1g.log; tail -2 gpurun_out/smoke_r1g.log
