timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or workspace or shard" 2>&1 | tail -1 > gpurun_out/t.txt
for c in cfg5 cfg2 cfg4; do timeout 60 python tools/gemm_probe.py $c 2>&1 | head -1 >> gpurun_out/t.txt; done
cat gpurun_out/t.txt
