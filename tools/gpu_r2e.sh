#!/bin/bash
mkdir -p gpurun_out
for cfg in "64,2048,2048,16,16 5:128:16:4" "64,2048,2048,64,64 5:128:64:4"; do
  set -- $cfg
  echo "=== trace none $1 plan $2"
  MBCI_LIB=trace timeout 120 python tools/trace_k5.py --op none --dtype bf16 --shape $1 --plan $2 --steps 8 2>&1 | sed -n 1,18p
done
