#!/bin/bash
# quick kernel-4 check: parity suite, then C2 / C3 timings with and without the tail split
timeout 900 python -m pytest tests/test_gpu_k4.py -q -x 2>&1 | tail -2
for ns in "" 1; do
  MBCI_T4_NO_SPLIT=$ns timeout 60 python tools/run_plan.py --plan 4:128:64:3 --iters 50 2>&1 | tail -1
  MBCI_T4_NO_SPLIT=$ns timeout 60 python tools/run_plan.py --plan 4:128:64:3 --shape 128,1024,1024,64,64 --dtype bf16 --iters 20 2>&1 | tail -1
done
MBCI_LIB=trace timeout 120 python tools/trace_chain4.py --plan 4:128:64:3 --tiles 8
