#!/bin/bash
./tools/microbench
for p in 128:64:2 64:64:2; do timeout 120 python tools/trace_chain.py --plan $p; done
