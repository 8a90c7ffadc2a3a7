timeout 30 python tools/shape_check.py 16 1024 1024; echo rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or workspace or shard" 2>&1 | tail -2
for m in 0 1; do ATOM_GEMM_PROBE_MODE=$m timeout 60 python tools/gemm_probe.py cfg5; done
ATOM_GEMM_TRACE=1 timeout 60 python tools/gemm_probe.py cfg5 > gpurun_out/trace5_g.log 2>&1
tail -5 gpurun_out/trace5_g.log
