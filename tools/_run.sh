for m in 0 2048 0 2048; do ATOM_GEMM_PROBE_MODE=$m timeout 60 python tools/gemm_probe.py cfg5 2>&1 | head -1; done > gpurun_out/t.txt
cat gpurun_out/t.txt
