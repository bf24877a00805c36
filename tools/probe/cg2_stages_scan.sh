# ncu: SM-pair GEMM ring depth (SMOE_CG2_STAGES builds) vs one-SM tiles, DRAM / clock / time
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum
for rep in 1 2; do
for cfg in mixtral qwen2_57b; do
  for v in "libsmoe.so 1" "libsmoe.so 2" "libsmoe_st4.so 2" "libsmoe_st5.so 2"; do
    set -- $v
    SMOE_LIB=paper_2503_04398_b200/$1 timeout 300 ncu --clock-control none --profile-from-start off -k "regex:grouped_gemm" -c 2 --metrics $M --csv python tools/probe/gemm_cg.py $2 $2 $cfg 16384 2>/dev/null | grep -v "^==" | sed "s/^/r$rep,$cfg,$1,cg$2,/"
  done
done
done
