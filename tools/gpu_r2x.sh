#!/bin/bash
run() { env $3 timeout 300 python bench.py --config $1 --steps 100 --warmup 5 --repeats 5 --sustain 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1 $2', round(d['ms_per_step']*1000,2), 'us', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do for c in C2 C6 C3; do
  run $c "current" ""
  run $c "prev2(before NONE change)" "MBCI_LIB=ab:libmbci_prev2.so"
  run $c "wait2" "MBCI_LIB=ab:libmbci_wait2.so"
done; done
