#!/bin/bash
# ring-depth sweep of kernel 5 on the plain chains (event-driven issuers, deferred P wait: flags 785)
mkdir -p gpurun_out
run() { MBCI_T5_FLAGS=$3 timeout 300 python bench.py --config $1 --plan $2 --steps 50 --warmup 5 --repeats 3 --sustain 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1 plan $2 flags $3', round(d['ms_per_step']*1000,2), 'us', d['clocks']['sm_mhz'], d['clocks']['reasons'], d['config']['plan'][:90])" || echo "$1 $2 failed"; }
for st in 4 5 6 7 8; do run C4-16 5:128:16:$st 785; done
for st in 4 5 6; do run C4-32 5:128:32:$st 785; done
for st in 3 4 5; do run C4-64 5:128:64:$st 785; done
for st in 4 5; do run C2 5:128:64:$st 785; done
for st in 4 5 6 7 8; do run C4-16 5:128:16:$st 17; done
