#!/bin/bash
# full GPU suite (k4 first), then the default bench line
timeout 1500 python -m pytest tests/test_gpu_k4.py -q 2>&1 | tail -5
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
