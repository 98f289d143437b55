#!/bin/bash
# bench lines for every config (default plans) -> gpurun_out/bench_all.jsonl
mkdir -p gpurun_out; : > gpurun_out/bench_all.jsonl
for c in C2 C1 C3 C4-16 C4-32 C4-64 C4-128 C5 C6; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --sustain 0.5 2>/dev/null >> gpurun_out/bench_all.jsonl
done
python - <<'PY'
import json
for l in open("gpurun_out/bench_all.jsonl"):
    try: j = json.loads(l)
    except Exception: continue
    r = j.get("roofline", {})
    print(f'{j["config"]["name"]:7s} {j["us_per_chain"]:9.2f} us  {j["value"]:8.1f} GB/s  frac {r.get("frac", 0):.3f}  tensor {r.get("tensor_tflops", 0):7.1f} TF/s  {j["clocks"]["sm_mhz"]} MHz {j["clocks"]["reasons"]}  e2e {j["e2e"]["value"]:.1f} GB/s  [{j["config"]["plan"][:48]}]')
PY
