M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum
for scale in 1.0 0.0156 0.0; do
  timeout 300 ncu --clock-control none --profile-from-start off -k "regex:grouped_gemm" -c 1 --metrics $M --csv \
    python tools/probe/gemm_single.py 1 8 4096 4096 28672 $scale 2>/dev/null | grep -v "^==" | sed "s/^/scale$scale,/"
done
