for m in 0 8192; do ATOM_GEMM_PROBE_MODE=$m timeout 60 python tools/gemm_probe.py cfg5 2>&1 | head -1; done > gpurun_out/t.txt
cat gpurun_out/t.txt
