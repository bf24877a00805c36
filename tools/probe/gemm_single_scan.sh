M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sector_hit_rate.pct
for shape in "1 4096 4096 28672" "8 4096 4096 28672" "1 8192 4096 28672" "1 4096 4096 2048"; do
  for cg in 1 2; do
    timeout 300 ncu --clock-control none --profile-from-start off -k "regex:grouped_gemm" -c 1 --metrics $M --csv \
      python tools/probe/gemm_single.py $cg $shape 2>/dev/null | grep -v "^==" | sed "s/^/cg${cg}_$(echo $shape | tr ' ' 'x'),/"
  done
done
