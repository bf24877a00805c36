M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum
for ut in 0 1; do
  for cg in 1 2; do
    SMOE_UNTILED_WEIGHTS=$ut timeout 300 ncu --clock-control none --profile-from-start off -k "regex:grouped_gemm" -c 2 --metrics $M --csv python tools/probe/gemm_cg.py $cg $cg mixtral 16384 2>/dev/null | grep -v "^==" | sed "s/^/ut${ut}_cg${cg},/"
  done
done
