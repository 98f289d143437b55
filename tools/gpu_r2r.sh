#!/bin/bash
MBCI_T5_FLAGS=3861 timeout 900 python -m pytest tests/test_gpu_persistent.py -q -x 2>&1 | tail -1
run() { env $3 timeout 300 python bench.py --config $1 --steps 100 --warmup 5 --repeats 5 --sustain 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1 $2', round(d['ms_per_step']*1000,2), 'us', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do for c in C2 C6 C4-16; do
  for f in 1809 3857 1813 3861; do run $c "flags $f" "MBCI_T5_FLAGS=$f"; done
done; done
