#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_causal.py tests/test_gpu_parity.py -q -x --timeout 120 > gpurun_out/pytest_causal.txt 2>&1; tail -3 gpurun_out/pytest_causal.txt
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/sanitize_synccheck.txt 2>&1; echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|Missing|err " gpurun_out/sanitize_synccheck.txt | head
