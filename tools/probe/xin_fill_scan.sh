M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for rep in 1 2; do for mt in 64 2048; do for fill in zero noise noise_xin noise_hmid; do
  timeout 300 ncu --clock-control none --profile-from-start off -k "regex:grouped_gemm" -c 1 --metrics $M --csv \
    python tools/probe/xin_fill.py 64 dsv2_lite $fill $mt 2>/dev/null | grep -v "^==" | sed "s/^/r$rep,mt$mt,$fill,/"
done; done; done
