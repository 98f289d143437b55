#!/bin/bash
# session 3: split-N suite first, then the whole GPU suite, then the default bench lines
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_splitn.py -x -q > gpurun_out/pytest_splitn.txt 2>&1; tail -15 gpurun_out/pytest_splitn.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
for c in C2 C6; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$c', round(d['ms_per_step']*1000,2), 'us', d['clocks'])"; done
