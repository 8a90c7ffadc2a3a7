timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/f_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/f_cfg5.log 2>&1
timeout 300 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/f_cfg2.log 2>&1
timeout 300 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/f_cfg4.log 2>&1
timeout 300 python bench.py --config cfg3_down --no-cpu-baseline > gpurun_out/f_cfg3d.log 2>&1
timeout 300 python bench.py --config cfg3_up --no-cpu-baseline > gpurun_out/f_cfg3u.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:w4a4_gemm -s 2 -c 1 -o gpurun_out/prof_final_cfg5 python tools/gemm_probe.py cfg5 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final_cfg5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/f_pytest.log gpurun_out/f_smoke.log
for f in f_cfg5 f_cfg2 f_cfg4 f_cfg3d f_cfg3u; do grep '^{' gpurun_out/$f.log | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$f', round(d['value'],1), round(d['ms_per_step']*1e3,1), d['kernels']['reorder_quantize']['us'], d['kernels']['w4a4_gemm']['us'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
