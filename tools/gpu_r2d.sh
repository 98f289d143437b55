#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_splitn.py -x -q > gpurun_out/pytest_splitn.txt 2>&1; tail -15 gpurun_out/pytest_splitn.txt
timeout 600 python bench.py --split-n 2 --steps 50 --warmup 5 > gpurun_out/bench_split2.json 2> gpurun_out/bench_split2.err; head -c 1500 gpurun_out/bench_split2.json; tail -3 gpurun_out/bench_split2.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
