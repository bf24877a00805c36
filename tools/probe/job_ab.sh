python -m pytest tests/test_gpu_layer.py tests/test_gpu_multiprocess.py -q -x -p no:cacheprovider 2>&1 | tail -2
bash tools/probe/build_ab.sh paper_2503_04398_b200/libsmoe_prev.so gpurun_out/prologue_ab.jsonl
