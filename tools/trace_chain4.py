"""Per-CTA timeline of the ping-pong kernel (kernel 4); needs MBCI_LIB=trace (libmbci_trace.so).
Prints, per flat tile g of CTA 0..n, the mean time (us from CTA start) of: S ready (slot 0/1),
P arrived at the issuer (slot 0/1), G2 issued (0/1), G1(g+1) issued (0/1), and per-unit epilogue."""
import sys, math, argparse, os
import numpy as np, torch
sys.path.insert(0, '.')
import mbci_inputs as gen
from paper_2506_22169_b200 import mbci
ap = argparse.ArgumentParser()
ap.add_argument("--plan", default="4:128:64:3")
ap.add_argument("--shape", default="96,512,512,64,64")
ap.add_argument("--dtype", default="f16")
ap.add_argument("--tiles", type=int, default=12)
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
S = 512
tr = torch.zeros(148 * S, dtype=torch.int64, device="cuda")
for i in range(50): ch.run(A, B, D, E)
torch.cuda.synchronize()
ch.set_trace(tr); ch.run(A, B, D, E); torch.cuda.synchronize(); ch.set_trace(None)
t = tr.cpu().numpy().reshape(148, S).astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
print(ch.describe(), "ctas", len(t))
print(f"kernel span {(t[:,3].max()-t0)/1000:.2f} us; CTA start spread {(t[:,0].max()-t0)/1000:.2f} us; "
      f"setup {np.mean(t[:,1]-t[:,0])/1000:.2f} us; CTA durations mean {np.mean(t[:,3]-t[:,0])/1000:.2f} max {np.max(t[:,3]-t[:,0])/1000:.2f}")
GHZ = float(os.environ.get("SM_GHZ", "1.965"))
def d(c):
    v = t[:, c]
    ok = v > 0
    return np.mean(v[ok] - t[ok, 4]) / GHZ / 1e3 if ok.mean() > 0.5 else float("nan")
names = ["S0", "S1", "max0", "max1", "Pst0", "Pst1", "Pseen0", "Pseen1", "G2_0", "G2_1", "G1_0", "G1_1",
         "Kwait", "Kland", "Pw0", "Pw1", "TMAiss"]
print("times in us from CTA start (clock64 / %.3f GHz)" % GHZ)
print("tile " + " ".join(f"{n:>6s}" for n in names) + "  sm0(max,exp) sm1(max,exp)")
for g in range(a.tiles):
    c = 8 + 16 * g
    row = [d(c + k) for k in range(16)] + [d(460 + g)]
    print(f"{g:4d} " + " ".join(f"{v:6.2f}" for v in row) +
          f"  {row[2]-row[0]:5.2f} {row[4]-row[2]:5.2f}  {row[3]-row[1]:5.2f} {row[5]-row[3]:5.2f}")
for u in range(4):
    print(f"unit {u}: epilogue o_full seen {d(490+4*u):.2f}  slot0 stored {d(490+4*u+1):.2f}  slot1 stored {d(490+4*u+2):.2f}")
if int(os.environ.get("MBCI_T4_DEBUG", "0")) & 8:
    print("latency probes (cycles, issue -> completion): G1_0 G1_1 G2_0 G2_1")
    for g in range(a.tiles):
        c = 8 + 16 * g
        v = [np.median(t[:, c + k][t[:, c + k] > 0]) if (t[:, c + k] > 0).mean() > 0.5 else float("nan") for k in (12, 13, 14, 15)]
        print(f"{g:4d} " + " ".join(f"{x:7.0f}" for x in v))
