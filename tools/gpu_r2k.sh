#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_chain_tc5 -s 3 -c 1 -o gpurun_out/r2_c3_k5 \
    python tools/ncu_one.py --config C3 --runs 5 > gpurun_out/r2_ncu_c3.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_c3_k5.ncu-rep > gpurun_out/r2_c3_k5_ncu_full.txt
cat gpurun_out/r2_c3_k5_ncu_full.txt | head -45
ncu -i gpurun_out/r2_c3_k5.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv, sys
rows = list(csv.reader(sys.stdin)); h = rows[0]
want = [k for k in h if any(s in k for s in ('pipe_xu', 'pipe_fma', 'pipe_alu', 'issue_active', 'inst_executed_pipe', 'sm__cycles_active.avg', 'smsp__cycles_active'))]
for k in want: print(k, rows[2][h.index(k)], rows[1][h.index(k)])
" > gpurun_out/r2_c3_k5_pipes.txt; cat gpurun_out/r2_c3_k5_pipes.txt | head -60
