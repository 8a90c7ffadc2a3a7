#!/usr/bin/env bash
# One GPU session: tests, bench lines, ncu launch list and full captures (run under gpurun).
# Usage: tools/gpu_round.sh TAG [configs...]
set -u
TAG=${1:-r01}; shift || true
CFGS=${@:-cfg5 cfg2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
python __graft_entry__.py > $OUT/build.log 2>&1
for c in $CFGS; do
  timeout -s KILL 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "bench $c rc=$?"; tail -c 1500 $OUT/bench_$c.json
done
# launch list (per-launch device times; cold-cache, serialised -> compare shares)
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $OUT/launches_cfg5.csv python bench.py --config cfg5 --steps 5 --warmup 3 \
  --no-e2e --no-cpu-baseline --spinup 0 > $OUT/launches_cfg5.log 2>&1
echo "ncu launches rc=$?"
for c in $CFGS; do
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:w4a4_gemm \
    -s 3 -c 1 -o $OUT/prof_gemm_$c python bench.py --config $c --steps 4 --warmup 3 --no-e2e \
    --no-cpu-baseline --spinup 0 > $OUT/prof_gemm_$c.log 2>&1
  echo "ncu gemm $c rc=$?"
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on \
    -k regex:reorder_quantize -s 3 -c 1 -o $OUT/prof_quant_$c python bench.py --config $c \
    --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --spinup 0 > $OUT/prof_quant_$c.log 2>&1
  echo "ncu quant $c rc=$?"
done
