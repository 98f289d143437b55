#!/bin/bash
# quick kernel-4 check: parity suite, bench (graph-timed) for the softmax and plain configs
timeout 900 python -m pytest tests/test_gpu_k4.py -q -x 2>&1 | tail -2
for c in C2 C3 C6 C4-16 C4-64 C4-128; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --sustain 0.2 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print(j['config']['name'], round(j['value'],1), 'GB/s', round(j['us_per_chain'],2), 'us', j['config']['plan'][:60])"
done
