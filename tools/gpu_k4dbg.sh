#!/bin/bash
for dbg in 1 3 5 2 4; do
 echo "=== MBCI_T4_DEBUG=$dbg"
 MBCI_T4_DEBUG=$dbg MBCI_LIB=trace MBCI_T4_EMU=3 timeout 120 python tools/trace_chain4.py --plan 4:128:64:3 --shape 128,1024,1024,64,64 --dtype bf16 --tiles 6 | head -12
done
