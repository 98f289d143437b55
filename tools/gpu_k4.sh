#!/bin/bash
# kernel-4 bring-up: parity tests, C2/C3 timings for k4 (MUFU-only and 3/8 polynomial) vs k0, trace.
timeout 900 python -m pytest tests/test_gpu_k4.py -x -q 2>&1 | tail -15
for e in 0 3; do
  for p in 4:128:64:3 4:128:64:4 4:128:64:6; do
    MBCI_T4_EMU=$e timeout 60 python tools/run_plan.py --plan $p --iters 20 2>&1 | tail -1
  done
  MBCI_T4_EMU=$e timeout 60 python tools/run_plan.py --plan 4:128:64:3 --shape 128,1024,1024,64,64 --dtype bf16 --iters 20 2>&1 | tail -1
  MBCI_T4_EMU=$e timeout 60 python tools/run_plan.py --plan 4:128:128:2 --shape 64,4096,4096,128,128 --dtype bf16 --iters 5 2>&1 | tail -1
done
timeout 60 python tools/run_plan.py --plan 0:64:64:2 --iters 20 2>&1 | tail -1
MBCI_LIB=trace MBCI_T4_EMU=3 timeout 120 python tools/trace_chain4.py --plan 4:128:64:3 --shape 128,1024,1024,64,64 --dtype bf16 --tiles 12
