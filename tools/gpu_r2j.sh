#!/bin/bash
# C2 / C6 / C3: turn variants on top of the session-3 defaults (785)
run() { env $3 timeout 300 python bench.py --config $1 --steps 100 --warmup 5 --repeats 5 --sustain 0.3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1 $2', round(d['ms_per_step']*1000,2), 'us', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do
for c in C2 C6; do
  run $c "flags785" "MBCI_T5_FLAGS=785"
  run $c "flags784-noturns" "MBCI_T5_FLAGS=784"
  run $c "flags769-handover0" "MBCI_T5_FLAGS=769"
  run $c "flags801-handover2" "MBCI_T5_FLAGS=801"
  run $c "flags817-handover3" "MBCI_T5_FLAGS=817"
  run $c "emu3" "MBCI_T4_EMU=3"
done; done
