# ncu scan of the down GEMM rasterisation (group_m) on one SM vs an SM pair (Mixtral 16K)
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum
for cg in 1 2; do
  for gm in 0 1 2 4 16 32 -1 -2 -4 -16; do
    SMOE_GROUP_M_DOWN=$gm timeout 300 ncu --clock-control none --profile-from-start off \
      -k "regex:grouped_gemm" -s 1 -c 1 --metrics $M --csv python tools/probe/gemm_cg.py 1 $cg mixtral 16384 \
      2>/dev/null | grep -v "^==" | sed "s/^/cg${cg}_gm${gm},/"
  done
done
