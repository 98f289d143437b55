"""Per-launch time vs batch (graph-timed, rotating inputs) for one shape: separates the fixed
per-launch cost from the per-unit cost.  usage: python tools/batch_sweep.py [--shape M,N,K,L]"""
import argparse, math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_22169_b200 import mbci
ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="512,512,64,64")
ap.add_argument("--dtype", default="f16")
ap.add_argument("--op", default="softmax")
ap.add_argument("--plan", default="")
ap.add_argument("--batches", default="1,2,4,12,24,48,96,148,192,296,384")
a = ap.parse_args()
M, N, K, L = map(int, a.shape.split(","))
dt = torch.float16 if a.dtype == "f16" else torch.bfloat16
res = []
for b in map(int, a.batches.split(",")):
    per = b * (M * K + N * K + N * L + M * L) * 2
    rot = max(2, math.ceil(300e6 / per))
    sets = [(torch.randn(b, M, K, device="cuda").to(dt), torch.randn(b, N, K, device="cuda").to(dt),
             torch.randn(b, N, L, device="cuda").to(dt), torch.empty(b, M, L, device="cuda", dtype=dt)) for _ in range(rot)]
    plan = None
    if a.plan:
        plan = mbci.mbci_plan_t(); plan.kernel, plan.BN, plan.TL, plan.stages = map(int, a.plan.split(":"))
    ch = mbci.Chain(b, M, N, K, L, a.dtype, a.op, 1 / math.sqrt(K), b_layout=1, plan=plan)
    st = torch.cuda.Stream()
    steps = 60
    with torch.cuda.stream(st):
        for i in range(5):
            A, B, D, E = sets[i % rot]; ch.run(A, B, D, E)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(steps):
            A, B, D, E = sets[i % rot]; ch.run(A, B, D, E)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        g.replay()
    e1.record(st); e1.synchronize()
    us = e0.elapsed_time(e1) / steps * 1e3
    res.append((b, us))
    print(f"batch {b:4d}: {us:8.2f} us/launch  {b * M / 256 / 148:.2f} pair-units/SM  [{ch.describe()[:40]}]", flush=True)
    del sets, g
