#!/bin/bash
# A/B: event-driven kernel-5 issuers (MBCI_T5_FLAGS bit 8) vs the in-order issuers
mkdir -p gpurun_out
MBCI_T5_FLAGS=273 timeout 900 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_splitn.py -q -x 2>&1 | tail -3
for rep in 1 2; do
for c in C2 C6 C4-16 C4-64 C3; do for f in 17 273; do
  MBCI_T5_FLAGS=$f timeout 300 python bench.py --config $c --steps 50 --warmup 5 --repeats 3 --sustain 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$c flags=$f', round(d['ms_per_step']*1000,2), 'us', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done; done
