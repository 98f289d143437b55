#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -8
bash tools/gpu_sweep.sh C2 0:128:64:2 0:128:64:3 0:64:64:2 0:64:64:4 2:64:64:2 2:64:64:3 2:64:64:4 3:128:64:2 3:128:64:3 3:128:64:4 3:128:64:6
bash tools/gpu_sweep.sh C6 0:64:64:2 2:64:64:3 3:128:64:3
bash tools/gpu_sweep.sh C3 0:64:64:2 2:64:64:3 3:128:64:3 3:128:64:4
bash tools/gpu_sweep.sh C4-64 0:128:64:2 2:64:64:3 3:128:64:3
bash tools/gpu_sweep.sh C5 0:128:128:2 3:128:128:2 3:128:128:3
