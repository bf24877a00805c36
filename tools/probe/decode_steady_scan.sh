M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for cfg in dsv2_lite mixtral qwen2_57b; do for warm in 0 1; do
  timeout 300 ncu --clock-control none --profile-from-start off -k "regex:grouped_gemm" -c 2 --metrics $M --csv \
    python tools/probe/decode_steady.py $cfg $warm 2>/dev/null | grep -v "^==" | sed "s/^/$cfg,warm$warm,/"
done; done
