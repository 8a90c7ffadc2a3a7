#!/usr/bin/env bash
# Round-end GPU session: tests, smoke, bench lines, config sweep, ncu launch list and full
# captures of the INT and MX GEMMs at cfg5 (run under gpurun).  Usage: tools/gpu_final.sh TAG
set -u
TAG=${1:-final}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
python __graft_entry__.py > $O/build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout -s KILL 600 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "bench rc=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_cfg5.json 2> $O/bench_reference.err; echo "ref rc=$?"
bash tools/sweep.sh $O/sweep.jsonl > $O/sweep.log 2>&1; echo "sweep done"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
  --spinup 0 --no-peak > $O/launches.log 2>&1; echo "ncu launches rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:w4a4_gemm \
  -s 3 -c 1 -o $O/prof_gemm_cfg5 python bench.py --steps 4 --warmup 3 --no-e2e \
  --no-cpu-baseline --spinup 0 --no-peak --no-mx > $O/prof_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:mx_gemm \
  -s 6 -c 2 -o $O/prof_mx_cfg5 python tools/mx_time.py "1024,28672,8192" > $O/prof_mx.log 2>&1; echo "ncu mx rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:reorder_quantize \
  -s 3 -c 1 -o $O/prof_quant_cfg5 python bench.py --steps 4 --warmup 3 --no-e2e \
  --no-cpu-baseline --spinup 0 --no-peak --no-mx > $O/prof_quant.log 2>&1; echo "ncu quant rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:decode_attention_kernel \
  -s 3 -c 1 -o $O/prof_kv python tools/kv_time.py "128,1024,32" > $O/prof_kv.log 2>&1; echo "ncu kv rc=$?"
