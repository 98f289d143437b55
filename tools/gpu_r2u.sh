#!/bin/bash
# per-chunk P store after an early p_free wait (MBCI_T5_FLAGS bit 12: 3857 -> 7953)
MBCI_T5_FLAGS=7953 timeout 900 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_causal.py -q -x 2>&1 | tail -2
run() { env $3 timeout 300 python bench.py --config $1 --steps 100 --warmup 5 --repeats 5 --sustain 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1 $2', round(d['ms_per_step']*1000,2), 'us', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do for c in C2 C6 C3; do
  run $c "flags 3857" "MBCI_T5_FLAGS=3857"
  run $c "flags 7953" "MBCI_T5_FLAGS=7953"
done; done
