#!/usr/bin/env bash
# BASELINE config sweep (L2-cold, device-timed): one bench JSON line per config into $1
OUT=${1:-gpurun_out/sweep.jsonl}; mkdir -p $(dirname $OUT); : > $OUT
for c in cfg1 cfg2 cfg4 cfg5 cfg3_up_m8 cfg3_up_m16 cfg3_up_m32 cfg3_up_m64 cfg3_up_m128 cfg3_up_m256 cfg3_up_m512 cfg3_up_m1024 cfg3_down_m8 cfg3_down_m16 cfg3_down_m32 cfg3_down_m64 cfg3_down_m128 cfg3_down_m256 cfg3_down_m512 cfg3_down_m1024; do
  timeout -s KILL 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-peak --no-kv 2>>${OUT%.jsonl}.err | tail -1 >> $OUT
  echo "$c rc=$?"
done
