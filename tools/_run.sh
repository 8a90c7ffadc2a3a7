timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b11.log 2>&1
tail -c 1500 gpurun_out/b11.log | python -c "import sys,json; l=[x for x in sys.stdin.read().splitlines() if x.startswith('{')]; d=json.loads(l[-1]); print(d['value'], d['kernels'])"
