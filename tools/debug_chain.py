"""Ad-hoc GPU diagnostics: S via D = I, error maps per case."""
import sys, math
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import mbci_inputs as gen, oracle
from gpu_helpers import run_chain, e_f64
from paper_2506_22169_b200 import mbci

def case(dtype, b, M, N, K, L, op, sc, b_layout=1, kind="int", eye=False, plan=None):
    inp = gen.make_chain_inputs(3, dtype, b, M, N, K, L, b_layout, kind=kind)
    if eye:
        e = np.eye(N, L)
        inp.D = gen._f64_to_storage(np.broadcast_to(e, (b, N, L)).ravel(), dtype).reshape(b, N, L)
    E, ch = run_chain(mbci, inp, op, sc, plan=plan)
    got = e_f64(E, dtype); ref = oracle.chain(inp, op, sc)
    err = oracle.row_max_error(got, ref)
    d = np.abs(got - ref)
    bad = np.argwhere(d > 1e-3 * (np.abs(ref).max() + 1e-9))
    print(f"{dtype} b={b} M={M} N={N} K={K} L={L} op={op} bl={b_layout} eye={eye}: err={err:.3e} bad={len(bad)} [{ch.describe()}]")
    if len(bad):
        rows = np.unique(bad[:, 1]); cols = np.unique(bad[:, 2]); bs = np.unique(bad[:, 0])
        print("   bad batches", bs[:10], "rows", rows[:10], "...", len(rows), "cols", cols[:20], len(cols))
        i = tuple(bad[0]); print("   first", i, "got", got[i], "ref", ref[i])
        if eye:
            bb, m = bad[0][0], bad[0][1]
            print("   got row", got[bb, m, :16]); print("   ref row", ref[bb, m, :16])
    return got, ref

for K in (16, 32, 64, 128):
    case("f16", 1, 128, 128, K, 128, "none", 1.0, eye=True)
for K in (16, 64):
    case("f16", 1, 128, 128, K, 128, "none", 1.0, eye=True, b_layout=0)
for K in (16, 64):
    case("f16", 1, 128, 128, K, 128, "softmax", 0.25, eye=True, kind="normal")
for K, L in ((16, 16), (16, 64), (64, 16), (32, 32), (128, 128), (128, 64), (64, 128)):
    case("f16", 2, 256, 256, K, L, "none", 1.0)
