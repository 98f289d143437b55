"""Per-slot timeline of the persistent kernel (kernel 2) via mbci_chain_set_trace."""
import sys, math, argparse
import numpy as np, torch
sys.path.insert(0, '.')
import mbci_inputs as gen
from paper_2506_22169_b200 import mbci
ap = argparse.ArgumentParser()
ap.add_argument("--plan", default="2:128:64:2")
ap.add_argument("--shape", default="96,512,512,64,64")
ap.add_argument("--dtype", default="f16")
ap.add_argument("--op", default="softmax")
a = ap.parse_args()
b, M, N, K, L = map(int, a.shape.split(","))
plan = mbci.mbci_plan_t()
plan.kernel, plan.BN, plan.TL, plan.stages = map(int, a.plan.split(":"))
inp = gen.make_chain_inputs(0, a.dtype, b, M, N, K, L, 1)
dt = torch.float16 if a.dtype == "f16" else torch.bfloat16
T = lambda x: torch.from_numpy(x.view(np.int16)).view(dt).cuda()
A, B, D = T(inp.A), T(inp.B), T(inp.D)
E = torch.empty(b, M, L, dtype=dt, device="cuda")
ch = mbci.Chain(b, M, N, K, L, a.dtype, a.op, 1 / math.sqrt(K), plan=plan)
nslots = 2 * 148
tr = torch.zeros(nslots * 256, dtype=torch.int64, device="cuda")
for i in range(5): ch.run(A, B, D, E)
ch.set_trace(tr); ch.run(A, B, D, E); torch.cuda.synchronize(); ch.set_trace(None)
t = tr.cpu().numpy().reshape(nslots, 256).astype(np.int64)
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
print(ch.describe(), "slots used", used.sum())
print(f"kernel span {(t[:,5].max()-t0)/1000:.2f} us; slot durations mean {np.mean(t[:,5]-t[:,0])/1000:.2f} us, max {np.max(t[:,5]-t[:,0])/1000:.2f}")
d = lambda c: np.mean(t[:, c] - t[:, 0]) / 1e3
print("setup %.2f" % d(1))
names = ["S rdy", "Sld w0", "Sld w1", "Sld w2", "Sld w3", "pfree", "P w0", "P w1", "P w2", "P w3", "M sfre", "M G1", "M pful", "M G2", "T B", "T D"]
print("tile " + " ".join(f"{n:>6s}" for n in names))
for g in range(8):
    c = 8 + 16 * g
    if (t[:, c] > 0).mean() < 0.5: break
    print(f"{g:4d} " + " ".join(f"{d(c+k):6.2f}" for k in range(16)))
en = np.sort((t[:, 5] - t0) / 1e3); print("slot end times (us): first/median/last", en[0], np.median(en), en[-1])
# slot 0 vs slot 1 separately for tile 2
for sl in (0, 1):
    tt = t[sl::2]
    c = 8 + 16 * 2
    print("slot", sl, "tile2:", " ".join(f"{np.mean(tt[:, c+k]-tt[:,0])/1e3:6.2f}" for k in range(16)))
print("MMA G1 issue detail: b_full ok, mma0..3 issued, after commit b_empty (us from slot start)")
for g in range(8):
    c = 128 + 8 * g
    print(f"{g:4d} " + " ".join(f"{d(c+k):6.2f}" for k in range(6)))
