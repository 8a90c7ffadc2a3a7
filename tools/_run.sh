timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or workspace or shard" 2>&1 | tail -1 > gpurun_out/t.txt
for s in 8,11008,4096 64,11008,4096 128,11008,4096 8,4096,11008 cfg2 16,1024,1024 cfg5; do timeout 60 python tools/gemm_probe.py $s 2>&1 | head -1; done >> gpurun_out/t.txt
cat gpurun_out/t.txt
