timeout 300 python bench.py > gpurun_out/b10_cfg5.log 2>&1
timeout 300 python bench.py --config cfg2 > gpurun_out/b10_cfg2.log 2>&1
timeout 300 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/b10_cfg4.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b10_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg5_v6.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b10_ncu.log 2>&1
for f in gpurun_out/b10_cfg5.log gpurun_out/b10_cfg2.log gpurun_out/b10_cfg4.log gpurun_out/b10_ref.log; do tail -c 250 $f; echo; done
