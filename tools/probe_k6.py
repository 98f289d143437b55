"""Exp-throughput probe of kernel 6 (trace build, MBCI_T4_DEBUG=256 [+512]): each softmax warp runs
its exponential block 64 times in the real kernel environment; prints exps/clk/SM.
usage: MBCI_LIB=trace MBCI_T4_DEBUG=256 MBCI_T6_FLAGS=1 python tools/probe_k6.py"""
import sys, os, math
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_22169_b200 import mbci
b, M, N, K, L = 296, 256, 128, 64, 64
plan = mbci.mbci_plan_t()
plan.kernel, plan.BN, plan.TL, plan.stages = 6, 128, 64, 4
A = torch.randn(b, M, K, device="cuda").half(); B = torch.randn(b, N, K, device="cuda").half()
D = torch.randn(b, N, L, device="cuda").half(); E = torch.empty(b, M, L, device="cuda").half()
ch = mbci.Chain(b, M, N, K, L, "f16", "softmax", 0.125, plan=plan)
tr = torch.zeros(148 * 512, dtype=torch.int64, device="cuda")
for _ in range(3): ch.run(A, B, D, E)
ch.set_trace(tr); ch.run(A, B, D, E); torch.cuda.synchronize(); ch.set_trace(None)
t = tr.cpu().numpy().reshape(148, 512)
cyc = t[:, 8:24].astype(np.float64)
per_sm = cyc.max(axis=1)
exps = 16 * 32 * 64 * 64
print(f"dbg={os.environ.get('MBCI_T4_DEBUG')} flags={os.environ.get('MBCI_T6_FLAGS')} emu={os.environ.get('MBCI_T4_EMU','2')}: "
      f"median SM {np.median(per_sm):.0f} cycles -> {exps / np.median(per_sm):.2f} exps/clk/SM "
      f"(warp cycles min {cyc.min():.0f} max {cyc.max():.0f})")
