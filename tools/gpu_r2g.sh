#!/bin/bash
# A/B: deferred P wait for the linear ops (MBCI_T5_FLAGS bit 9) on top of the event-driven issuers
mkdir -p gpurun_out
MBCI_T5_FLAGS=785 timeout 900 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_ops.py -q -x 2>&1 | tail -2
for c in C4-16 C4-64 C2 C6; do for f in 17 785; do
  MBCI_T5_FLAGS=$f timeout 300 python bench.py --config $c --steps 50 --warmup 5 --repeats 3 --sustain 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$c flags=$f', round(d['ms_per_step']*1000,2), 'us', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
for f in 785; do
  echo "=== trace C4-16 flags $f"
  MBCI_T5_FLAGS=$f MBCI_LIB=trace timeout 120 python tools/trace_k5.py --op none --dtype bf16 --shape 64,2048,2048,16,16 --plan 5:128:16:4 --steps 8 2>&1 | sed -n 1,14p
done
