#!/bin/bash
MBCI_T4_FLAGS=1024 timeout 900 python -m pytest tests/test_gpu_persistent.py -q -x -k "k4 or kernel4 or 4" 2>&1 | tail -1
run() { env $3 timeout 600 python bench.py --config $1 --steps $4 --warmup 3 --repeats 3 --sustain 0.5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1 $2', round(d['ms_per_step']*1000,2), 'us', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do
  run C4-128 "t4flags0" "MBCI_T4_FLAGS=0" 50; run C4-128 "t4flags1024" "MBCI_T4_FLAGS=1024" 50
  run C5 "t4flags0" "MBCI_T4_FLAGS=0" 5; run C5 "t4flags1024" "MBCI_T4_FLAGS=1024" 5
done
