#!/bin/bash
# round-2 (session 3) probe: sanity bench + smoke, then k5 phase timeline in free-running vs pipeline
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; head -c 400 gpurun_out/bench_c2.json; echo
for e in 0 2; do
  echo "=== pipeline EMU=$e"; MBCI_T4_EMU=$e timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step']*1000, 'us')"
done
for d in 0 128 134 6; do
  echo "=== trace MBCI_T4_DEBUG=$d"
  MBCI_LIB=trace MBCI_T4_DEBUG=$d timeout 120 python tools/trace_k5.py --steps 7 2>&1 | sed -n 1,14p
done
