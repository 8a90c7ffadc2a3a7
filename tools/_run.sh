timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/t9_pytest.log
for c in cfg5 cfg2 cfg4 cfg3_up cfg3_down cfg1; do timeout 60 python tools/gemm_probe.py $c; done > gpurun_out/t9_probe.log 2>&1
timeout 300 python bench.py > gpurun_out/t9_bench.log 2>&1
timeout 300 python bench.py --config cfg2 > gpurun_out/t9_bench2.log 2>&1
cat gpurun_out/t9_pytest.log gpurun_out/t9_probe.log; tail -c 300 gpurun_out/t9_bench.log
