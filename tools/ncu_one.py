"""Run one config's default (or forced) plan eagerly a few times — a target for `ncu -k ... -c 1`.
usage: python tools/ncu_one.py [--config C2] [--plan K:BN:TL:stages] [--runs 8]"""
import argparse, math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mbci_inputs as gen
from paper_2506_22169_b200 import mbci
import bench
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--plan", default="")
ap.add_argument("--runs", type=int, default=8)
a = ap.parse_args()
dtype, b, M, N, K, L, op, *_ = bench.CONFIGS[a.config]
bl = 1 if op == "softmax" else 0
sig = (1.0, 1.0, 1.0) if op == "softmax" else (1.0, 1 / math.sqrt(K), 1 / math.sqrt(N))
inp = gen.make_chain_inputs(0, dtype, b, M, N, K, L, bl, sigmas=sig)
tdt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[dtype]
T = lambda x: torch.from_numpy(x.view(np.int32 if dtype == "f32" else np.int16)).view(tdt).cuda()
A, B, D = T(inp.A), T(inp.B), T(inp.D)
E = torch.empty(b, M, L, dtype=tdt, device="cuda")
plan = None
if a.plan:
    plan = mbci.mbci_plan_t()
    plan.kernel, plan.BN, plan.TL, plan.stages = map(int, a.plan.split(":"))
ch = mbci.Chain(b, M, N, K, L, dtype, op, 1 / math.sqrt(K) if op == "softmax" else 1.0, b_layout=bl, plan=plan)
print(ch.describe(), flush=True)
for _ in range(a.runs):
    ch.run(A, B, D, E)
torch.cuda.synchronize()
