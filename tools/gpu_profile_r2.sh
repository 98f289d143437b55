#!/bin/bash
# round-2 evidence for the default C2 kernel: launch list of the bench command, one full ncu capture
# with L2 write sectors (E's write volume stays in L2 at kernel end), summaries into gpurun_out/
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_c2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sustain 0 > gpurun_out/r2_launches_bench.log 2>&1
ncu --set full --metrics lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --import-source on -k regex:k_chain_tc5 -s 5 -c 1 -o gpurun_out/r2_c2_k5 \
    python tools/ncu_one.py --config C2 --runs 8 > gpurun_out/r2_ncu_k5.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_c2_k5.ncu-rep > gpurun_out/r2_c2_k5_ncu_full.txt
ncu -i gpurun_out/r2_c2_k5.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv, sys
rows = list(csv.reader(sys.stdin)); h = rows[0]
for r in rows[2:]:
    for k in ('lts__t_sectors_op_write.sum', 'lts__t_sectors_op_read.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum'):
        if k in h: print(k, r[h.index(k)], rows[1][h.index(k)])
" > gpurun_out/r2_c2_k5_traffic.txt
ncu -i gpurun_out/r2_c2_k5.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_c2_k5_src.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/r2_c2_k5_src.csv > gpurun_out/r2_c2_k5_stalls.txt 2>&1
