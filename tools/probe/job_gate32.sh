python -m pytest tests/test_gpu_layer.py tests/test_gpu_fuzz.py tests/test_gpu_multiprocess.py -q -x -p no:cacheprovider 2>&1 | tail -2
out=gpurun_out/gate_quarters_ab.jsonl; : > $out
for rep in 1 2; do
  for lib in paper_2503_04398_b200/libsmoe.so paper_2503_04398_b200/libsmoe_prev.so; do
    for t in 64 512 16384; do
      SMOE_LIB=$PWD/$lib timeout 300 python tools/stage_probe.py --stages gate --tokens $t | sed "s#}\$#, \"lib\": \"$lib\"}#" >> $out
    done
  done
done
bash tools/probe/build_ab.sh paper_2503_04398_b200/libsmoe_prev.so gpurun_out/gate_quarters_layer_ab.jsonl 64,512,16384
