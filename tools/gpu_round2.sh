#!/bin/bash
./tools/microbench
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider 2>&1 | grep -E "^(FAILED|ERROR)|passed|failed" | head -30
for p in "" 128:64:2 128:64:3 128:64:4 64:64:2 64:64:3 64:64:4 64:32:3 128:32:3; do
  echo "plan=$p $(timeout 120 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --sustain 0.2 ${p:+--plan $p} | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(round(j["value"],1), "GB/s", round(j["us_per_chain"],2), "us", j["config"]["plan"])')"
done
