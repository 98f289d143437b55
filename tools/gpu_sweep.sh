#!/bin/bash
# Plan sweep on one config: every kernel family x stages, plus tune=1.  Usage: gpu_sweep.sh CONFIG PLAN...
cfg=$1; shift
mkdir -p gpurun_out
for p in "$@"; do
  r=$(timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline --sustain 0.1 --plan $p 2>&1 | tail -1)
  echo "$cfg plan=$p $(echo "$r" | python -c 'import sys,json
try:
  j=json.loads(sys.stdin.read()); print(round(j["value"],1), "GB/s", round(j["us_per_chain"],2), "us", round(j["roofline"]["tensor_frac"],3))
except Exception as e: print("ERR", e)')"
done
