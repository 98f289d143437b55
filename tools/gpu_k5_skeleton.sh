#!/bin/bash
# kernel-5 skeleton decomposition (trace build): per debug mode / flags, one traced launch of C2
mkdir -p gpurun_out
for d in ${DBG:-0 1 6 7 16 23 64}; do for f in ${FLAGS:-17}; do
  echo "=== MBCI_T4_DEBUG=$d MBCI_T5_FLAGS=$f"
  MBCI_LIB=trace MBCI_T4_DEBUG=$d MBCI_T5_FLAGS=$f timeout 120 python tools/trace_k5.py --steps 7 ${ARGS:-} 2>&1 | sed -n 1,12p
done; done
