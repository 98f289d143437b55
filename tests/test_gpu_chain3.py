"""Three-contraction chains E3 = op2(op(A·B)·D)·F (mbci_chain3_*, R20)
against the fp64 oracle (oracle.chain3, pinned in test_oracle_pins.py): the MLP-style chain
(GELU between every contraction pair), attention with a following projection, masks, large K
(live k loop) and H cut into chunks on the grid; integer chains bit for bit."""
import math

import numpy as np
import pytest
import torch

import mbci_inputs as gen
import oracle
from gpu_helpers import e_bits, e_f64, rn_bits, to_dev

pytestmark = pytest.mark.gpu

BUDGET = {"f16": 4e-3, "bf16": 1.5e-2}


@pytest.fixture(scope="module")
def mbci():
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    from paper_2506_22169_b200 import mbci as m
    return m


def make_F(seed, dtype, b, L, H, kind="normal", sigma=1.0):
    return gen.make_chain_inputs(seed, dtype, b, L, 1, H, 1, 1, kind=kind, sigmas=(sigma, 1.0, 1.0)).A   # [b, L, H]


def run3(mbci, inp, F, H, op, scale, op2, scale2, valid_len=None, causal=False):
    ch = mbci.Chain3(inp.batch, inp.M, inp.N, inp.K, inp.L, H, inp.dtype, op, scale, op2, scale2,
                     mask=valid_len is not None, causal=causal, b_layout=inp.b_layout)
    A, B, D, Fd = (to_dev(x, inp.dtype) for x in (inp.A, inp.B, inp.D, F))
    E = torch.full((inp.batch, inp.M, H), float("nan"), dtype=A.dtype, device="cuda")
    vl = None if valid_len is None else torch.from_numpy(np.asarray(valid_len, np.int32)).cuda()
    ch.run(A, B, D, Fd, E, vl)
    torch.cuda.synchronize()
    return E, ch


@pytest.mark.parametrize("dtype,op,op2", [("bf16", "gelu", "gelu"), ("f16", "softmax", "none"),
                                          ("bf16", "relu", "scale"), ("f16", "none", "relu")])
@pytest.mark.parametrize("M,N,K,L,H", [(256, 384, 64, 64, 128), (300, 200, 48, 40, 96), (128, 512, 128, 128, 256)])
def test_chain3_parity(mbci, dtype, op, op2, M, N, K, L, H):
    sig = (1.0, 1.0, 1.0) if op == "softmax" else (1.0, 1.0 / math.sqrt(K), 1.0 / math.sqrt(N))
    inp = gen.make_chain_inputs(900 + K + H, dtype, 3, M, N, K, L, 1, sigmas=sig)
    F = make_F(901 + H, dtype, 3, L, H, sigma=1.0 / math.sqrt(L))
    sc = 1.0 / math.sqrt(K) if op == "softmax" else 1.0
    E, ch = run3(mbci, inp, F, H, op, sc, op2, 0.8)
    got = e_f64(E, dtype)
    ref = oracle.chain3(inp, F, H, op, sc, op2, 0.8)
    assert np.all(np.isfinite(got))
    err = oracle.row_max_error(got, ref)
    assert err <= BUDGET[dtype], (err, ch.plan().BN, ch.plan().TL)


def test_chain3_masks_and_large_K(mbci):
    inp = gen.make_chain_inputs(910, "bf16", 4, 256, 512, 256, 64, 1, sigmas=(1.0, 1.0, 1.0))
    F = make_F(911, "bf16", 4, 64, 192, sigma=0.125)
    vl = np.array([512, 1, 0, 300], dtype=np.int32)
    E, _ = run3(mbci, inp, F, 192, "softmax", 1 / 16, "gelu", 1.0, valid_len=vl, causal=True)
    ref = oracle.chain3(inp, F, 192, "softmax", 1 / 16, "gelu", 1.0, valid_len=vl, causal=True)
    assert oracle.row_max_error(e_f64(E, "bf16"), ref) <= BUDGET["bf16"]
    assert torch.all(E[2] == 0)


def test_chain3_integer_bitwise(mbci):
    """Integer A, B, D, F in [-2, 2], NONE / NONE and RELU: |C| <= 128, |O| <= 2^15 ... kept exact in
    fp16 by K = L = 16 (|C| <= 64, |O| <= 64·2·N <= 2048 with N = 16), H = 64."""
    inp = gen.make_chain_inputs(920, "f16", 2, 256, 16, 16, 16, 0, kind="int")
    F = make_F(921, "f16", 2, 16, 64, kind="int")
    for op2 in ("none", "relu"):
        E, _ = run3(mbci, inp, F, 64, "none", 1.0, op2, 1.0)
        assert np.array_equal(e_bits(E), rn_bits(oracle.chain3(inp, F, 64, "none", 1.0, op2, 1.0), "f16"))


def test_chain3_rejects_unsupported(mbci):
    with pytest.raises(mbci.MbciError):
        mbci.Chain3(1, 128, 128, 64, 192, 64, "f16", "softmax", 0.125, "none")   # L > 128
    with pytest.raises(mbci.MbciError):
        mbci.Chain3(1, 128, 128, 64, 64, 60, "f16", "softmax", 0.125, "none")    # H not a multiple of 8
    with pytest.raises(mbci.MbciError):
        mbci.Chain3(1, 128, 128, 64, 64, 64, "f16", "softmax", 0.125, "softmax")  # op2 softmax
