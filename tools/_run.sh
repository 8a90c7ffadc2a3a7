for m in 0 4096; do ATOM_GEMM_PROBE_MODE=$m timeout 60 python tools/gemm_probe.py cfg5 > /tmp/o.txt 2>&1; head -1 /tmp/o.txt; done
timeout 60 python tools/gemm_probe.py cfg2 2>&1 | head -1
ATOM_GEMM_TRACE=1 timeout 60 python tools/gemm_probe.py cfg5 > gpurun_out/trace5_p.log 2>&1
grep -A45 "^g " gpurun_out/trace5_p.log | tail -5
