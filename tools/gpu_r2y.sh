#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_parity.py tests/test_gpu_ops.py tests/test_gpu_splitn.py tests/test_gpu_causal.py -q -x 2>&1 | tail -1
run() { env $3 timeout 300 python bench.py --config $1 --steps 100 --warmup 5 --repeats 5 --sustain 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1 $2', round(d['ms_per_step']*1000,2), 'us', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do for c in C2 C6 C3 C4-16 C4-64; do
  run $c "split-instantiations" ""
  run $c "prev2" "MBCI_LIB=ab:libmbci_prev2.so"
done; done
