"""Run one chain shape with a forced plan a few times (for ncu captures and quick timing).
usage: python tools/run_plan.py --plan K:BN:TL:stages --shape b,M,N,K,L [--dtype f16] [--iters 5]"""
import sys, math, argparse
import numpy as np, torch
sys.path.insert(0, '.')
import mbci_inputs as gen
from paper_2506_22169_b200 import mbci
ap = argparse.ArgumentParser()
ap.add_argument("--plan", default="")
ap.add_argument("--shape", default="96,512,512,64,64")
ap.add_argument("--dtype", default="f16")
ap.add_argument("--op", default="softmax")
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
b, M, N, K, L = map(int, a.shape.split(","))
plan = None
if a.plan:
    plan = mbci.mbci_plan_t()
    plan.kernel, plan.BN, plan.TL, plan.stages = map(int, a.plan.split(":"))
bl = 1 if a.op == "softmax" else 0
inp = gen.make_chain_inputs(0, a.dtype, b, M, N, K, L, bl)
dt = torch.float16 if a.dtype == "f16" else torch.bfloat16
T = lambda x: torch.from_numpy(x.view(np.int16)).view(dt).cuda()
A, B, D = T(inp.A), T(inp.B), T(inp.D)
E = torch.empty(b, M, L, dtype=dt, device="cuda")
ch = mbci.Chain(b, M, N, K, L, a.dtype, a.op, 1 / math.sqrt(K), b_layout=bl, plan=plan)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(2): ch.run(A, B, D, E)
e0.record()
for i in range(a.iters): ch.run(A, B, D, E)
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) / a.iters * 1e3
print(f"{ch.describe()}  {us:.2f} us/run  {2.0*b*M*N*(K+L)/us/1e6:.1f} TFLOP/s  {b*M*N/us/1e6/148:.3f} Gexp/s/SM")
