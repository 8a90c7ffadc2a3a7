timeout 30 python tools/shape_check.py 16 1024 1024 > gpurun_out/t.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or workspace or shard or rmsnorm_fused" 2>&1 | tail -1 >> gpurun_out/t.txt
for s in cfg5 cfg2 8,11008,4096 64,11008,4096 cfg4 cfg3_down; do timeout 60 python tools/gemm_probe.py $s 2>&1 | head -1; done >> gpurun_out/t.txt
cat gpurun_out/t.txt
