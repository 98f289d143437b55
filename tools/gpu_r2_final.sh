#!/bin/bash
# round-2 (session 3) evidence with the final defaults: GPU suite, smoke, bench lines, ncu
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; head -c 300 gpurun_out/bench_c2.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; head -c 200 gpurun_out/bench_ref.json; echo
STEPS=50 bash tools/gpu_bench_all.sh > gpurun_out/bench_all_summary.txt 2>&1; cat gpurun_out/bench_all_summary.txt
bash tools/gpu_profile_r2.sh; cat gpurun_out/r2_c2_k5_traffic.txt; head -30 gpurun_out/r2_c2_k5_ncu_full.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_merge -c 3 --csv \
    --log-file gpurun_out/r2_merge_ncu.csv python bench.py --split-n 2 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --sustain 0 > /dev/null 2>&1
tail -4 gpurun_out/r2_merge_ncu.csv
