#!/bin/bash
echo "=== trace C6"; MBCI_LIB=trace timeout 120 python tools/trace_k5.py --shape 96,256,256,64,64 --steps 3 2>&1 | sed -n 1,30p
echo "=== trace C2"; MBCI_LIB=trace timeout 120 python tools/trace_k5.py --steps 7 2>&1 | sed -n 1,16p
