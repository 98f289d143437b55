#!/bin/bash
# A/B of run-time variants: graph-timed bench lines per (config, env assignment).
# usage: tools/gpu_ab.sh "ENV1 ENV2 ..." "C2 C3 ..." [pytest -k filter for tests/test_gpu_persistent.py]
#   each ENV is a comma-separated list of VAR=value (or "-" for the defaults)
mkdir -p gpurun_out
EV=${1:--}; CF=${2:-C2}; PT=${3:-}
if [ -n "$PT" ]; then timeout 900 python -m pytest tests/test_gpu_persistent.py -q -x -k "$PT" 2>&1 | tail -3; fi
for c in $CF; do for e in $EV; do
  envs=""; [ "$e" != "-" ] && envs=$(echo "$e" | tr ',' ' ')
  r=$(env $envs timeout 300 python bench.py --config $c ${PLAN:+--plan $PLAN} --steps 50 --warmup 5 --no-cpu-baseline --sustain 0.3 2>/dev/null)
  echo "$r" | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('$c $e', round(j['us_per_chain'],2), 'us', j['clocks']['sm_mhz'], j['clocks']['reasons'])" 2>/dev/null || echo "$c $e FAILED"
done; done
