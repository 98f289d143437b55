#!/bin/bash
export MBCI_LIB=trace
echo "=== k0 BN128 C2"; timeout 120 python tools/trace_chain.py --plan 128:64:2
echo "=== k0 BN64 C2"; timeout 120 python tools/trace_chain.py --plan 64:64:2
echo "=== k0 BN128 long N"; timeout 120 python tools/trace_chain.py --plan 128:64:2 --shape 148,128,4096,64,64
echo "=== k3 C2"; WARM_S=1 timeout 120 python tools/trace_chain3.py --plan 3:128:64:3
echo "=== k3 long N"; WARM_S=1 timeout 120 python tools/trace_chain3.py --plan 3:128:64:3 --shape 148,256,4096,64,64
