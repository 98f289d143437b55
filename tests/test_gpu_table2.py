"""Parity of the live k loop and of L chunking on PAPER.md Table II's GEMM-chain
shapes: G1-G3 (K = 64, H = 64/128/256), G4-G6 (K = 256/512/1024, H = 256),
G7-G12 (K = H = 128, M up to 2048, batch up to 8), through the C ABI against the fp64 oracle.

K > 128 runs kernel 0 with A and B streamed in 64-column chunks (TcParams::kc); L > 128 runs
kernel 0 with <= 128-column h chunks bound to the grid (S recomputed per chunk).
Integer chains whose products and sums are exact in fp16 / fp32 must match RN(oracle) bit for bit.
"""
import math

import numpy as np
import pytest
import torch

import mbci_inputs as gen
import oracle
from gpu_helpers import e_bits, e_f64, rn_bits, run_chain

pytestmark = pytest.mark.gpu

BUDGET = {"f16": 4e-3, "bf16": 1.5e-2}

TABLE2 = {   # name: (batch, M, N, K, H)
    "G1": (1, 512, 256, 64, 64), "G2": (1, 512, 256, 64, 128), "G3": (1, 512, 256, 64, 256),
    "G4": (1, 512, 512, 256, 256), "G5": (1, 512, 512, 512, 256), "G6": (1, 512, 512, 1024, 256),
    "G7": (1, 512, 512, 128, 128), "G8": (1, 1024, 512, 128, 128), "G9": (1, 2048, 512, 128, 128),
    "G10": (1, 1024, 1024, 128, 128), "G11": (4, 1024, 1024, 128, 128), "G12": (8, 1024, 1024, 128, 128),
}


@pytest.fixture(scope="module")
def mbci():
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    from paper_2506_22169_b200 import mbci as m
    return m


def _plain_inputs(seed, dtype, b, M, N, K, L, b_layout=0):
    return gen.make_chain_inputs(seed, dtype, b, M, N, K, L, b_layout,
                                 sigmas=(1.0, 1.0 / math.sqrt(K), 1.0 / math.sqrt(N)))


@pytest.mark.parametrize("name", sorted(TABLE2))
def test_table2_gemm_chain(mbci, name):
    b, M, N, K, L = TABLE2[name]
    inp = _plain_inputs(400 + K + L, "f16", b, M, N, K, L)
    rows = np.stack([np.repeat(np.arange(b), 64), np.tile(np.arange(0, M, M // 64), b)], axis=1).astype(np.int64)
    E, ch = run_chain(mbci, inp, "none", 1.0)
    if K > 128 or L > 128:
        assert ch.plan().kernel == 0, ch.describe()
    err = oracle.row_max_error(e_f64(E, "f16")[rows[:, 0], rows[:, 1]], oracle.chain(inp, "none", 1.0, rows=rows))
    assert err <= BUDGET["f16"], (err, ch.describe())


@pytest.mark.parametrize("K,L,b_layout", [(256, 64, 1), (512, 128, 0), (1024, 64, 1), (64, 256, 1), (200, 200, 0),
                                          (300, 136, 1)])
def test_softmax_large_K_or_L(mbci, K, L, b_layout):
    inp = gen.make_chain_inputs(500 + K, "bf16", 2, 384, 640, K, L, b_layout)
    E, ch = run_chain(mbci, inp, "softmax", 1.0 / math.sqrt(K))
    err = oracle.row_max_error(e_f64(E, "bf16"), oracle.chain(inp, "softmax", 1.0 / math.sqrt(K)))
    assert err <= BUDGET["bf16"], (err, ch.describe())


@pytest.mark.parametrize("K,L,b_layout", [(256, 192, 0), (512, 64, 1), (384, 256, 1), (136, 40, 0)])
def test_integer_chain_bitwise_large_K_L(mbci, K, L, b_layout):
    """|C| <= 4K <= 2048 is exact in fp16 and every fp32 partial sum of E is an exact integer."""
    inp = gen.make_chain_inputs(600 + K, "f16", 2, 300, 384, K, L, b_layout, kind="int")
    for op, sc in (("none", 1.0), ("scale", 0.5)):
        E, ch = run_chain(mbci, inp, op, sc)
        assert np.array_equal(e_bits(E), rn_bits(oracle.chain(inp, op, sc), "f16")), ch.describe()


def test_every_plan_agrees_large_K(mbci):
    """Every legal plan of a G4-like shape (live k loop; BN 64 / 128, TL 16..128, stages)."""
    b, M, N, K, L = 1, 256, 512, 256, 256
    inp = _plain_inputs(7, "bf16", b, M, N, K, L)
    ref = oracle.chain(inp, "none", 1.0)
    st, plans = mbci.plan_enumerate(mbci.make_desc(b, M, N, K, L, "bf16", "none", 1.0, b_layout=0))
    assert st == 0 and len(plans) >= 4 and all(p.kernel == 0 for p in plans)
    for p in plans[:12]:
        E, ch = run_chain(mbci, inp, "none", 1.0, plan=p)
        assert oracle.row_max_error(e_f64(E, "bf16"), ref) <= BUDGET["bf16"], ch.describe()
