timeout 300 ncu --set full --import-source on --clock-control none -k regex:reorder_quantize -s 5 -c 1 -o gpurun_out/prof_q5b python tools/gemm_probe.py cfg5 > /dev/null 2>&1
