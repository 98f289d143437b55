"""Same chain shape in fp16 and bf16 through the ABI (CUDA events, graph of `steps` launches, rotating
inputs) — isolates the cost of the 16-bit type (the P / E conversions) at a fixed shape.
usage: python tools/dtype_ab.py [--shape b,M,N,K,L] [--op softmax]"""
import argparse, math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mbci_inputs as gen
from paper_2506_22169_b200 import mbci
ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="96,512,512,64,64")
ap.add_argument("--op", default="softmax")
ap.add_argument("--steps", type=int, default=100)
a = ap.parse_args()
b, M, N, K, L = map(int, a.shape.split(","))
bl = 1 if a.op == "softmax" else 0
for dt in ("f16", "bf16"):
    tdt = torch.float16 if dt == "f16" else torch.bfloat16
    inp = gen.make_chain_inputs(0, dt, b, M, N, K, L, bl, sigmas=(1, 1, 1) if a.op == "softmax" else (1, 1 / math.sqrt(K), 1 / math.sqrt(N)))
    T = lambda x: torch.from_numpy(x.view(np.int16)).view(tdt).cuda()
    sets = [(T(inp.A), T(inp.B), T(inp.D), torch.empty(b, M, L, dtype=tdt, device="cuda")) for _ in range(8)]
    ch = mbci.Chain(b, M, N, K, L, dt, a.op, 1 / math.sqrt(K) if a.op == "softmax" else 1.0, b_layout=bl)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(10):
            ch.run(*sets[i % 8], stream=st)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(a.steps):
            ch.run(*sets[i % 8], stream=st)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            g.replay()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / a.steps * 1e3)
    print(f"{dt:5s} {a.op} {a.shape}: {sorted(ts)[2]:.2f} us  [{ch.describe()[:60]}]", flush=True)
    ch.close()
