#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_chain_tc5 -s 3 -c 1 -o gpurun_out/r2_c416_k5 \
    python tools/ncu_one.py --config C4-16 --runs 5 > gpurun_out/r2_ncu_c416.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_c416_k5.ncu-rep > gpurun_out/r2_c416_k5_ncu_full.txt
head -45 gpurun_out/r2_c416_k5_ncu_full.txt
ncu -i gpurun_out/r2_c416_k5.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_c416_src.csv 2>/dev/null
