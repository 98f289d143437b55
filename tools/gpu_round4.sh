#!/bin/bash
python - <<'PY'
import sys, math, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import mbci_inputs as gen, oracle
from gpu_helpers import run_chain, e_f64
from paper_2506_22169_b200 import mbci
def plan(k, bn, tl, st):
    p = mbci.mbci_plan_t(); p.kernel, p.BN, p.TL, p.stages = k, bn, tl, st; return p
cases = [("f16", 2, 256, 256, 64, 64, "softmax", 1), ("f16", 96, 512, 512, 64, 64, "softmax", 1),
         ("bf16", 3, 300, 333, 64, 40, "softmax", 1), ("bf16", 4, 256, 512, 64, 64, "none", 1),
         ("f16", 5, 128, 1000, 48, 64, "softmax", 0), ("bf16", 2, 256, 512, 128, 128, "softmax", 1)]
for dt, b, M, N, K, L, op, bl in cases:
    sig = (1,1,1) if op == "softmax" else (1, 1/math.sqrt(K), 1/math.sqrt(N))
    inp = gen.make_chain_inputs(1, dt, b, M, N, K, L, bl, sigmas=sig)
    ref = oracle.chain(inp, op, 1/math.sqrt(K))
    for pl in ([plan(2, 128, 64, 2), plan(2, 64, 64, 2), plan(2, 128, 64, 3)] if L <= 64 else [plan(2, 64, 128, 2)]):
        try:
            E, ch = run_chain(mbci, inp, op, 1/math.sqrt(K), plan=pl)
            err = oracle.row_max_error(e_f64(E, dt), ref)
            print(f"{dt} {b}x{M}x{N}x{K}x{L} {op} bl={bl}: err={err:.3e}  [{ch.describe()}]", flush=True)
        except Exception as e:
            print("FAIL", dt, b, M, N, K, L, op, pl.BN, pl.TL, pl.stages, repr(e)[:300], flush=True)
PY
for p in 2:128:64:2 2:64:64:2 2:128:64:3 0:128:64:2; do
  echo "plan=$p $(timeout 120 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --sustain 0.2 --plan $p | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(round(j["value"],1), "GB/s", round(j["us_per_chain"],2), "us", j["config"]["plan"])')"
done
