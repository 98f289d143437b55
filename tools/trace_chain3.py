"""Per-CTA timeline of the two-Q-tile kernel (kernel 3); needs MBCI_LIB=trace."""
import sys, math, argparse
import numpy as np, torch
sys.path.insert(0, '.')
import mbci_inputs as gen
from paper_2506_22169_b200 import mbci
ap = argparse.ArgumentParser()
ap.add_argument("--plan", default="3:128:64:3")
ap.add_argument("--shape", default="96,512,512,64,64")
ap.add_argument("--dtype", default="f16")
a = ap.parse_args()
b, M, N, K, L = map(int, a.shape.split(","))
plan = mbci.mbci_plan_t()
plan.kernel, plan.BN, plan.TL, plan.stages = map(int, a.plan.split(":"))
inp = gen.make_chain_inputs(0, a.dtype, b, M, N, K, L, 1)
dt = torch.float16 if a.dtype == "f16" else torch.bfloat16
T = lambda x: torch.from_numpy(x.view(np.int16)).view(dt).cuda()
A, B, D = T(inp.A), T(inp.B), T(inp.D)
E = torch.empty(b, M, L, dtype=dt, device="cuda")
ch = mbci.Chain(b, M, N, K, L, a.dtype, "softmax", 1 / math.sqrt(K), plan=plan)
tr = torch.zeros(148 * 256, dtype=torch.int64, device="cuda")
import time
t_end = time.time() + float(__import__("os").environ.get("WARM_S", "0"))
while True:
    for i in range(50): ch.run(A, B, D, E)
    torch.cuda.synchronize()
    if time.time() >= t_end: break
ch.set_trace(tr); ch.run(A, B, D, E); torch.cuda.synchronize(); ch.set_trace(None)
t = tr.cpu().numpy().reshape(148, 256).astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
print(ch.describe(), "ctas", len(t))
print(f"kernel span {(t[:,5].max()-t0)/1000:.2f} us; CTA durations mean {np.mean(t[:,5]-t[:,0])/1000:.2f}")
d = lambda c: np.mean(t[:, c] - t[:, 0]) / 1e3
mhz = (t[:, 7] - t[:, 6]) / ((t[:, 5] - t[:, 0]) / 1e3)
print("effective SM clock during the kernel (MHz): min %.0f median %.0f max %.0f" % (mhz.min(), np.median(mhz), mhz.max()))
names = ["S0 rdy", "P0", "S1 rdy", "P1", "M dful", "M p0", "M G2G1_0", "M p1", "M G2G1_1", "-", "T B", "T D"]
print("tile " + " ".join(f"{n:>8s}" for n in names))
for g in range(8):
    c = 8 + 16 * g
    if (t[:, c] > 0).mean() < 0.5: break
    print(f"{g:4d} " + " ".join(f"{d(c+k):8.2f}" for k in range(12)))
