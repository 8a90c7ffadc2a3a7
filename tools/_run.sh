timeout 30 python tools/shape_check.py 16 1024 1024; echo rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or workspace or shard" 2>&1 | tail -1
for c in cfg5 cfg2; do timeout 60 python tools/gemm_probe.py $c 2>&1 | head -1; done
