python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
bash tools/probe/pdl_ab.sh gpurun_out/pdl_ab2.jsonl
