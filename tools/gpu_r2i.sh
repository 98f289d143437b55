#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_splitn.py -q -x 2>&1 | tail -2
timeout 300 python bench.py --split-n 2 --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('split2', round(d['ms_per_step']*1000,2), 'us')"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum --clock-control none -k regex:k_merge -c 3 --csv \
    --log-file gpurun_out/r2_merge_ncu.csv python bench.py --split-n 2 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --sustain 0 > /dev/null 2>&1
grep -o '"[a-z_]*__[a-z_.]*","[a-z]*","[0-9.]*"' gpurun_out/r2_merge_ncu.csv | tail -8
