M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum
for rep in 1 2; do for cfg in mixtral qwen2_57b; do for lib in libsmoe_base.so libsmoe_cssc.so libsmoe_csall.so; do
  SMOE_LIB=paper_2503_04398_b200/$lib timeout 300 ncu --clock-control none --profile-from-start off -k "regex:grouped_gemm|combine" -c 3 --metrics $M --csv python tools/probe/gemm_cg.py 1 2 $cfg 16384 2>/dev/null | grep -v "^==" | sed "s/^/r$rep,$cfg,$lib,/"
done; done; done
