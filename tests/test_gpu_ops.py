"""Elementwise inter-ops RELU and GELU (R19; the MLP-style chain E = act(s·A·B)·D) on
every kernel family, through the C ABI, against the fp64 oracle (pinned in test_oracle_pins.py):
16-bit within the 16-bit budget, fp32 (kernels 7 and 1) within 1e-5, RELU on integer chains bit
for bit (max(C, 0) of an exact integer C is exact), and the plain-chain half items."""
import math

import numpy as np
import pytest
import torch

import mbci_inputs as gen
import oracle
from gpu_helpers import e_bits, e_f64, rn_bits, run_chain

pytestmark = pytest.mark.gpu

BUDGET = {"f16": 4e-3, "bf16": 1.5e-2, "f32": 1e-5}


@pytest.fixture(scope="module")
def mbci():
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    from paper_2506_22169_b200 import mbci as m
    return m


def plan(mbci, k, L=64):
    p = mbci.mbci_plan_t()
    p.kernel, p.BN, p.TL, p.stages = k, 128, L, {5: 4, 6: 4, 4: 3, 0: 2}.get(k, 1)
    return p


def _inputs(seed, dtype, b, M, N, K, L, b_layout=1):
    return gen.make_chain_inputs(seed, dtype, b, M, N, K, L, b_layout,
                                 sigmas=(1.0, 1.0 / math.sqrt(K), 1.0 / math.sqrt(N)))


@pytest.mark.parametrize("op", ["relu", "gelu"])
@pytest.mark.parametrize("kernel,dtype", [(5, "f16"), (6, "bf16"), (4, "bf16"), (0, "f16"), (None, "bf16")])
def test_activation_16bit(mbci, op, kernel, dtype):
    inp = _inputs(800 + (kernel or 9), dtype, 4, 384, 512, 64, 64)
    E, ch = run_chain(mbci, inp, op, 1.5, plan=None if kernel is None else plan(mbci, kernel))
    if kernel is not None:
        assert ch.plan().kernel == kernel, ch.describe()
    err = oracle.row_max_error(e_f64(E, dtype), oracle.chain(inp, op, 1.5))
    assert err <= BUDGET[dtype], (err, ch.describe())


@pytest.mark.parametrize("op", ["relu", "gelu"])
@pytest.mark.parametrize("kernel", [7, 1])
def test_activation_fp32(mbci, op, kernel):
    inp = _inputs(810, "f32", 2, 200, 260, 32, 48)
    p = mbci.mbci_plan_t()
    p.kernel = kernel
    E, ch = run_chain(mbci, inp, op, 0.8, plan=p)
    assert ch.plan().kernel == kernel
    err = oracle.row_max_error(e_f64(E, "f32"), oracle.chain(inp, op, 0.8))
    assert err <= BUDGET["f32"], (err, ch.describe())


@pytest.mark.parametrize("kernel", [5, 4, 0])
def test_relu_integer_chain_bitwise(mbci, kernel):
    inp = gen.make_chain_inputs(820, "f16", 3, 256, 384, 64, 64, 1, kind="int")
    E, ch = run_chain(mbci, inp, "relu", 1.0, plan=plan(mbci, kernel))
    assert np.array_equal(e_bits(E), rn_bits(oracle.chain(inp, "relu", 1.0), "f16")), ch.describe()


@pytest.mark.parametrize("op", ["relu", "gelu"])
def test_activation_half_items_and_default_scale(mbci, op):
    """156 x 512 rows: the last pair units run as half items (slot partials summed); scale NaN
    selects 1 for the activations (R19)."""
    b, M, N, K = 156, 512, 512, 64
    inp = _inputs(830, "bf16", b, M, N, K, K)
    E, ch = run_chain(mbci, inp, op, float("nan"), plan=plan(mbci, 5))
    rows = np.concatenate([np.stack([np.full(M, b - 1), np.arange(M)], axis=1),
                           np.stack([np.arange(b), (np.arange(b) * 37) % M], axis=1)]).astype(np.int64)
    ref = oracle.chain(inp, op, 1.0, rows=rows)
    err = oracle.row_max_error(e_f64(E, "bf16")[rows[:, 0], rows[:, 1]], ref)
    assert err <= BUDGET["bf16"], (err, ch.describe())
