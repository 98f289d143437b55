#!/bin/bash
# Round-1 re-entry session: gpu tests, smoke, bench, ncu launch list + full capture of the top kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nproc; lscpu | grep 'Model name'
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt; cat gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
bash tools/gpu_bench_round.sh > gpurun_out/bench_round.log 2>&1
tail -30 gpurun_out/bench_round.log
