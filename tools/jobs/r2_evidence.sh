#!/bin/bash
# Round-2 evidence on one B200: GPU suite, smoke, bench line (both arms),
# per-step launch list and ncu --set full of the layer kernels of the timed step.
#   TAG=r2a tools/jobs/r2_evidence.sh      (run under gpurun)
cd "$(dirname "$0")/../.."
TAG=${TAG:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider -x > gpurun_out/gpu_tests_$TAG.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_$TAG.log
  tail -3 gpurun_out/gpu_tests_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo rc=$? >> gpurun_out/smoke_$TAG.log
  tail -2 gpurun_out/smoke_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
tail -c 400 gpurun_out/bench_$TAG.json
if [ -z "$SKIP_REF" ]; then
  timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo ref rc=$?
fi
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
  --no-dsmoe --no-decode > /dev/null 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:grouped_gemm|gate_tc|srs_kernel|combine_sag|dispatch_kernel" \
  -s 6 -c 6 -f -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu \
  --no-dsmoe --no-decode > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_full.ncu-rep --page details --csv > gpurun_out/${TAG}_full_details.csv 2>/dev/null
ls -la gpurun_out | tail -20
