#!/bin/bash
# A/B of two in-tree builds (SMOE_LIB): layer latency eager / graph, output hashes.
# usage: build_ab.sh <alt.so> <out.jsonl> [tokens]
alt=$1; out=$2; toks=${3:-64,512,2048,16384}
: > $out
for rep in 1 2; do
  for cfg in mixtral dsv2_lite qwen2_57b; do
    for lib in paper_2503_04398_b200/libsmoe.so $alt; do
      SMOE_LIB=$PWD/$lib timeout 300 python tools/latency.py --config $cfg --tokens $toks --reps 40 \
        | sed "s#}\$#, \"lib\": \"$lib\"}#" >> $out 2>>${out%.jsonl}.err
    done
  done
done
