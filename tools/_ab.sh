# A/B: time every ab/*.so variant on the given configs (interleaved, 2 rounds)
{
for r in 1 2; do
for v in ab/*.so; do
  cp $v paper_2310_19102_b200/libatom.so
  for c in "$@"; do echo -n "$(basename $v) "; PROBE_REPS=${PROBE_REPS:-1} timeout 120 python tools/gemm_probe.py $c 2>&1 | grep gemm; done
done
done
} > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
