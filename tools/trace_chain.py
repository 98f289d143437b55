"""Per-CTA timeline of the tensor-core kernel (mbci_chain_set_trace) for one config/plan."""
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
a = ap.parse_args()
b, M, N, K, L = map(int, a.shape.split(","))
plan = None
if a.plan:
    plan = mbci.mbci_plan_t(); plan.kernel = 0
    plan.BN, plan.TL, plan.stages = map(int, a.plan.split(":"))
inp = gen.make_chain_inputs(0, a.dtype, b, M, N, K, L, 1)
dt = torch.float16 if a.dtype == "f16" else torch.bfloat16
T = lambda x: torch.from_numpy(x.view(np.int16)).view(dt).cuda()
A, B, D = T(inp.A), T(inp.B), T(inp.D)
E = torch.empty(b, M, L, dtype=dt, device="cuda")
ch = mbci.Chain(b, M, N, K, L, a.dtype, a.op, 1 / math.sqrt(K), plan=plan)
nb = ch.plan().n_block
S = 128
tr = torch.zeros(nb * S, dtype=torch.int64, device="cuda")
for i in range(5): ch.run(A, B, D, E)
ch.set_trace(tr); ch.run(A, B, D, E); torch.cuda.synchronize(); ch.set_trace(None)
t = tr.cpu().numpy().reshape(nb, S).astype(np.int64)
t0 = t[:, 0].min()
print(ch.describe())
nt = (N + ch.plan().BN - 1) // ch.plan().BN
print(f"kernel span {(t[:,5].max()-t0)/1000:.2f} us; CTA durations mean {np.mean(t[:,5]-t[:,0])/1000:.2f} us")
d = lambda c: np.mean(t[:, c] - t[:, 0]) / 1e3
print("mean per-CTA phase (us from CTA start): setup %.2f  A %.2f" % (d(1), d(3)))
names = ["S ready", "S loaded", "max", "exp", "P arrive", "G1 issued", "G2 issued"]
print("tile  " + "  ".join(f"{n:>9s}" for n in names))
for j in range(min(nt, 16)):
    print(f"{j:4d}  " + "  ".join(f"{d(8 + 7*j + k):9.2f}" for k in range(7)))
print("  epi start %.2f  end %.2f" % (d(4), d(5)))
st = np.sort((t[:, 0] - t0) / 1e3); print("CTA start times (us): first/median/last", st[0], np.median(st), st[-1])
en = np.sort((t[:, 5] - t0) / 1e3); print("CTA end times (us): first/median/last", en[0], np.median(en), en[-1])
sm = t[:, 2]
print("CTAs per SM: max", np.bincount(sm).max(), "min", np.bincount(sm, minlength=148).min())
