"""Causal-mask parity (R18): key n visible to query row m iff n <= m
(top-left aligned), alone and combined with key padding, on every kernel family that takes it —
kernels 5 and 4 (persistent: the pair's slot 0 runs the pair's last key tile fully masked), kernel
0 (incl. the live k loop and h chunks), kernel 7 (fp32, 3xTF32) and kernel 1 (CUDA cores) —
against the fp64 oracle (itself pinned to torch SDPA is_causal, tests/test_oracle_pins.py)."""
import math

import numpy as np
import pytest
import torch

import mbci_inputs as gen
import oracle
from gpu_helpers import e_f64, run_chain

pytestmark = pytest.mark.gpu

BUDGET = {"f16": 4e-3, "bf16": 1.5e-2, "f32": 1e-5}


@pytest.fixture(scope="module")
def mbci():
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    from paper_2506_22169_b200 import mbci as m
    return m


def plan(mbci, k, L, K=64):
    p = mbci.mbci_plan_t()
    p.kernel, p.BN, p.TL = k, 128, max(16, (L + 15) // 16 * 16)
    p.stages = {5: 2 if K > 64 else 4, 4: 3 if L <= 64 else 2, 0: 2}.get(k, 1)
    if k == 0:
        p.TL = min(p.TL, 128)
    return p


def check(mbci, inp, scale, kernel=None, valid_len=None):
    pl = None if kernel is None else plan(mbci, kernel, inp.L, inp.K)
    E, ch = run_chain(mbci, inp, "softmax", scale, valid_len=valid_len, plan=pl, causal=True)
    if kernel is not None:
        assert ch.plan().kernel == kernel, ch.describe()
    got = e_f64(E, inp.dtype)
    ref = oracle.chain(inp, "softmax", scale, valid_len=valid_len, causal=True)
    assert np.all(np.isfinite(got))
    err = oracle.row_max_error(got, ref)
    assert err <= BUDGET[inp.dtype], (err, ch.describe())
    return E, ch


@pytest.mark.parametrize("kernel", [5, 4, 0])
@pytest.mark.parametrize("M,N", [(512, 512), (384, 512), (512, 300), (130, 129)])
def test_causal_16bit(mbci, kernel, M, N):
    inp = gen.make_chain_inputs(700 + M + N, "f16", 4, M, N, 64, 64, 1)
    E, ch = check(mbci, inp, 0.125, kernel)
    D = gen.bits_to_f64_numpy(inp.D, "f16")
    assert np.array_equal(e_f64(E, "f16")[:, 0, :], D[:, 0, :])   # row 0 sees key 0 only: P = 1


@pytest.mark.parametrize("kernel", [5, 4, 0])
def test_causal_with_key_padding(mbci, kernel):
    b = 6
    inp = gen.make_chain_inputs(31, "bf16", b, 512, 512, 64, 64, 1, sigmas=(2.0, 2.0, 1.0))
    vl = np.array([512, 1, 0, 200, 128, 511], dtype=np.int32)
    E, _ = check(mbci, inp, 0.125, kernel, valid_len=vl)
    assert torch.all(E[2] == 0)


def test_causal_default_plan_and_many_units(mbci):
    """Default plan (kernel 5) over 300 pair units with one key-tile count per pair."""
    inp = gen.make_chain_inputs(33, "f16", 150, 512, 512, 64, 64, 1)
    rows = np.stack([np.arange(150), (np.arange(150) * 101) % 512], axis=1).astype(np.int64)
    E, ch = run_chain(mbci, inp, "softmax", 0.125, causal=True)
    assert ch.plan().kernel == 5, ch.describe()
    ref = oracle.chain(inp, "softmax", 0.125, rows=rows, causal=True)
    err = oracle.row_max_error(e_f64(E, "f16")[rows[:, 0], rows[:, 1]], ref)
    assert err <= BUDGET["f16"], err


@pytest.mark.parametrize("K,L", [(256, 64), (64, 256), (128, 128)])
def test_causal_kernel0_large_dims(mbci, K, L):
    inp = gen.make_chain_inputs(40 + K + L, "bf16", 2, 384, 384, K, L, 1)
    check(mbci, inp, 1.0 / math.sqrt(K))


def test_causal_fp32_kernels(mbci):
    inp = gen.make_chain_inputs(41, "f32", 2, 200, 260, 32, 48, 1)
    check(mbci, inp, 0.2, 7)
    check(mbci, inp, 0.2, 1)
    check(mbci, gen.make_chain_inputs(42, "bf16", 2, 3, 5, 3, 3, 0), 0.5, 1)   # TMA-illegal rows: kernel 1


def test_causal_rejects_non_softmax(mbci):
    with pytest.raises(mbci.MbciError):
        mbci.Chain(1, 128, 128, 64, 64, "f16", "none", 1.0, causal=True)
