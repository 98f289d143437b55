#!/bin/bash
# One GPU session: GPU tests, bench (C2 + other configs), reference arm, ncu launch list + full capture.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err
cat gpurun_out/bench_c2.json
rm -f gpurun_out/bench_other.json
for c in C6 C3 C4-16 C4-64 C4-128; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --sustain 0.3 >> gpurun_out/bench_other.json 2>> gpurun_out/bench_other.err
done
timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --sustain 0.3 >> gpurun_out/bench_other.json 2>> gpurun_out/bench_other.err
cat gpurun_out/bench_other.json | python -c "import sys,json; [print(j['config']['name'], round(j['value'],1), round(j['us_per_chain'],2), round(j['roofline']['tensor_frac'],3), j['config']['plan']) for j in map(json.loads, sys.stdin)]"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --sustain 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_tc -s 5 -c 1 -o gpurun_out/prof_c2 -f python bench.py --steps 8 --warmup 3 --no-cpu-baseline --sustain 0 > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
ls gpurun_out
