#!/usr/bin/env bash
# time every ab/*.so on the given configs (dev A/B, one process per variant and config)
for c in ${CFGS:-cfg5}; do for so in ab/*.so; do
  case $so in *probe*) continue;; esac
  timeout -s KILL 60 python tools/ab_gemm.py $so $c 5 ${WHAT:-gemm} 2>&1 | tail -1
done; done
