"""Model-fidelity study on B200 (§VI-E, Figs. 10-11):
for GEMM-chain / attention shapes, time EVERY legal plan of the selector and report
  * Spearman rank correlation of the measured time with the paper's t_estm (Eqs. 2-5) and with the
    B200 score t_b200, and the regret of each model's top-1 (measured time / measured optimum);
  * the SMEM estimate of Eq. 1 (one tile per staged tensor) against the exact dynamic shared memory
    of the plan (the kernels multi-buffer, so Eq. 1 under-counts by the pipeline depth);
  * PAPER.md Algorithm 1 (tune = 2, GPU-timed) on the same shape: rounds, measurements and the
    regret of its plan against the exhaustive optimum.
usage: python tools/model_study.py [--out profiles/r2_model_study.json]"""
import argparse, json, math, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_22169_b200 import mbci

SHAPES = {   # name: (batch, M, N, K, L, dtype, op, b_layout)
    "G1": (1, 512, 256, 64, 64, "f16", "none", 0), "G2": (1, 512, 256, 64, 128, "f16", "none", 0),
    "G7": (1, 512, 512, 128, 128, "f16", "none", 0), "G8": (1, 1024, 512, 128, 128, "f16", "none", 0),
    "G9": (1, 2048, 512, 128, 128, "f16", "none", 0), "G10": (1, 1024, 1024, 128, 128, "f16", "none", 0),
    "G11": (4, 1024, 1024, 128, 128, "f16", "none", 0), "G12": (8, 1024, 1024, 128, 128, "f16", "none", 0),
    "C2": (96, 512, 512, 64, 64, "f16", "softmax", 1), "C6": (96, 256, 256, 64, 64, "f16", "softmax", 1),
    "C4-64": (64, 2048, 2048, 64, 64, "bf16", "none", 0),
}
TD = {"f16": torch.float16, "bf16": torch.bfloat16}


def rank(x):
    r = np.empty(len(x))
    r[np.argsort(x)] = np.arange(len(x))
    return r


def spearman(a, b):
    if len(a) < 3:
        return float("nan")
    return float(np.corrcoef(rank(np.asarray(a)), rank(np.asarray(b)))[0, 1])


def time_plan(b, M, N, K, L, dt, op, bl, plan, bufs, reps=20):
    ch = mbci.Chain(b, M, N, K, L, dt, op, 0.125 if op == "softmax" else 1.0, b_layout=bl, plan=plan)
    A, B, D, E = bufs
    for _ in range(3):
        ch.run(A, B, D, E)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(st)
        ch.run(A, B, D, E)
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    ch.close()
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/model_study.json")
    ap.add_argument("--shapes", default=",".join(SHAPES))
    a = ap.parse_args()
    res = {}
    for name in a.shapes.split(","):
        b, M, N, K, L, dt, op, bl = SHAPES[name]
        d = mbci.make_desc(b, M, N, K, L, dt, op, 0.125 if op == "softmax" else 1.0, b_layout=bl)
        st, plans = mbci.plan_enumerate(d)
        g = torch.Generator(device="cuda").manual_seed(0)
        A = torch.randn(b, M, K, device="cuda", generator=g).to(TD[dt])
        B = (torch.randn(b, K, N, device="cuda", generator=g) if bl == 0 else
             torch.randn(b, N, K, device="cuda", generator=g)).to(TD[dt]) / math.sqrt(K)
        D = torch.randn(b, N, L, device="cuda", generator=g).to(TD[dt]) / math.sqrt(N)
        E = torch.empty(b, M, L, device="cuda", dtype=TD[dt])
        rows = []
        for p in plans:
            t = time_plan(b, M, N, K, L, dt, op, bl, p, (A, B, D, E))
            s = 2
            dch = -(-p.TL // 64)
            shm_eq1 = (p.BM * p.TK + p.TK * p.BN + p.BN * p.TL) * s   # Eq. 1: one tile per staged tensor
            rows.append(dict(kernel=p.kernel, BN=p.BN, TL=p.TL, stages=p.stages, t_meas=t, t_estm=p.t_estm,
                             t_b200=p.t_b200, smem=p.smem_bytes, shm_eq1=shm_eq1))
        tm = np.array([r["t_meas"] for r in rows])
        opt = float(tm.min())
        te = np.array([r["t_estm"] for r in rows])
        tb = np.array([r["t_b200"] for r in rows])
        t0 = time.time()
        ch = mbci.Chain(b, M, N, K, L, dt, op, 0.125 if op == "softmax" else 1.0, b_layout=bl, tune=2)
        t_search = time.time() - t0
        r_, m_ = ctypes_stats(ch)
        sp = ch.plan()
        t_alg1 = time_plan(b, M, N, K, L, dt, op, bl, sp, (A, B, D, E))
        ch.close()
        res[name] = dict(
            plans=len(rows), t_opt=opt,
            spearman_estm=spearman(te, tm), spearman_b200=spearman(tb, tm),
            regret_estm=float(tm[np.argmin(te)] / opt), regret_b200=float(tm[np.argmin(tb)] / opt),
            eq1_over_actual=float(np.median([r["shm_eq1"] / r["smem"] for r in rows])),
            alg1=dict(rounds=r_, measurements=m_, seconds=t_search, plan=[sp.kernel, sp.BN, sp.TL, sp.stages],
                      regret=float(t_alg1 / opt)),
            rows=rows)
        x = res[name]
        print(f"{name:6s} plans {x['plans']:3d}  opt {opt * 1e6:8.2f} us  spearman estm {x['spearman_estm']:+.2f} "
              f"b200 {x['spearman_b200']:+.2f}  regret estm {x['regret_estm']:.2f} b200 {x['regret_b200']:.2f}  "
              f"Eq1/actual SMEM {x['eq1_over_actual']:.2f}  Alg1: {r_} rounds {m_} meas regret {x['alg1']['regret']:.2f} "
              f"({t_search:.1f} s)", flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


def ctypes_stats(ch):
    import ctypes
    r, m = ctypes.c_int32(), ctypes.c_int32()
    mbci.check(mbci.mbci_chain_search_stats(ch.h, ctypes.byref(r), ctypes.byref(m)), "search_stats")
    return r.value, m.value


if __name__ == "__main__":
    main()
