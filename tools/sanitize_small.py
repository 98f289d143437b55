"""Small runs of every kernel family for compute-sanitizer (racecheck / synccheck / memcheck):
kernels 4, 5, 6 (persistent, with half items), 0 (incl. the live k loop), 7 (fp32 3xTF32), 1."""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mbci_inputs as gen
import oracle
from paper_2506_22169_b200 import mbci
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from gpu_helpers import run_chain, e_f64

def plan(k, BN=128, TL=64, st=4):
    p = mbci.mbci_plan_t(); p.kernel, p.BN, p.TL, p.stages = k, BN, TL, st; return p

cases = [
    ("k5 half items", gen.make_chain_inputs(1, "f16", 6, 512, 512, 64, 64, 1), "softmax", 0.125, plan(5)),
    ("k6", gen.make_chain_inputs(2, "f16", 4, 256, 384, 64, 64, 1), "softmax", 0.125, plan(6)),
    ("k4", gen.make_chain_inputs(3, "bf16", 4, 256, 384, 64, 64, 1), "softmax", 0.125, plan(4, st=3)),
    ("k0", gen.make_chain_inputs(4, "f16", 2, 256, 384, 64, 64, 1), "softmax", 0.125, plan(0, st=2)),
    ("k0 live k", gen.make_chain_inputs(5, "f16", 1, 256, 256, 256, 64, 0), "none", 1.0, None),
    ("k7 fp32", gen.make_chain_inputs(6, "f32", 2, 130, 200, 16, 16, 1), "softmax", 0.25, None),
    ("k1", gen.make_chain_inputs(7, "f16", 2, 3, 5, 3, 3, 0), "softmax", 0.5, None),
]
for name, inp, op, sc, pl in cases:
    E, ch = run_chain(mbci, inp, op, sc, plan=pl)
    err = oracle.row_max_error(e_f64(E, inp.dtype), oracle.chain(inp, op, sc))
    print(f"{name}: {ch.describe()[:40]} err {err:.2e}")
