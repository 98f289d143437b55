"""Parity of the persistent ping-pong kernels with the fp64 oracle: kernel 4 (chain_tc4.cuh, P
aliasing S, any L <= 128), kernel 5 (chain_tc5.cuh, separate P buffers, L <= 64) and kernel 6
(chain_tc6.cuh, kernel 5 with every score row split over two softmax warps), each forced through
mbci_chain_create_with_plan so every case runs that kernel (cases with L > 64 skip kernels 5, 6).

Covers: both B layouts and dtypes, head dims 16..128 (d = 128 single-buffers Q), ragged M
(a pair unit whose second 128-row tile is entirely past M), ragged N and K/L not multiples of
16, key padding (0, 1, partial-tile and full lengths, mixed within one launch so CTAs see
units with different tile counts), the lazy-rescale path, negative / zero scale, rows summing
to one, more units than CTAs (Q buffers, o_free and the K/V ring cycle many times), both
exponential paths (MUFU only, and 3/8 of the pairs on the FMA-pipe polynomial), run-to-run
bitwise determinism, and strided operands.
"""
import math
import os

import numpy as np
import pytest
import torch

import mbci_inputs as gen
import oracle
from gpu_helpers import e_bits, e_f64, rn_bits, run_chain, to_dev

pytestmark = pytest.mark.gpu

TOL = {"f16": 2e-2, "bf16": 2e-2}
BUDGET = {"f16": 4e-3, "bf16": 1.5e-2}


@pytest.fixture(scope="module")
def mbci():
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    from paper_2506_22169_b200 import mbci as m
    return m


@pytest.fixture(params=["0", "2", "3"], ids=["mufu", "poly2of8", "poly3of8"])
def emu(request, monkeypatch):
    monkeypatch.setenv("MBCI_T4_EMU", request.param)
    return request.param


_KERN = {"k": 4}


@pytest.fixture(autouse=True, params=[4, 5, 6], ids=["k4", "k5", "k6"])
def kern(request):
    _KERN["k"] = request.param
    yield request.param


def k4_plan(mbci, L, stages=None, K=64):
    """Plan of the kernel under test (fixture `kern`) for head dims K, L."""
    k = _KERN["k"]
    if k >= 5 and L > 64:
        pytest.skip("kernels 5 and 6 keep S_0, S_1, P_0, P_1, O_0, O_1 in TMEM: L <= 64")
    if stages is None:   # kernel 4, TL <= 64: three S buffers need a 3-deep ring; d = 128 fits only 2
        stages = 3 if L <= 64 else 2
        if k >= 5 and K > 64:   # two 64-column Q / K chunks and the E staging: a 2-deep ring fits
            stages = 2
    p = mbci.mbci_plan_t()
    p.kernel, p.BN, p.TL, p.stages = k, 128, max(16, (L + 15) // 16 * 16), stages
    return p


def check4(mbci, inp, scale, valid_len=None, stages=None, rows=None):
    E, ch = run_chain(mbci, inp, "softmax", scale, valid_len, plan=k4_plan(mbci, inp.L, stages, inp.K))
    assert ch.plan().kernel == _KERN["k"], ch.describe()
    got = e_f64(E, inp.dtype)
    if rows is not None:
        ref = oracle.chain(inp, "softmax", scale, valid_len=valid_len, rows=rows)
        got = got[rows[:, 0], rows[:, 1]]
    else:
        ref = oracle.chain(inp, "softmax", scale, valid_len=valid_len)
    assert np.all(np.isfinite(got)), "non-finite output"
    err = oracle.row_max_error(got, ref)
    assert err <= BUDGET[inp.dtype], (err, ch.describe())
    return E, ch


@pytest.mark.parametrize("dtype,b_layout", [("f16", 1), ("bf16", 1), ("f16", 0), ("bf16", 0)])
def test_k4_bert_base_slice(mbci, emu, dtype, b_layout):
    inp = gen.make_chain_inputs(1, dtype, 8, 512, 512, 64, 64, b_layout)
    check4(mbci, inp, 0.125)


@pytest.mark.parametrize("K,L", [(16, 16), (32, 64), (64, 128), (128, 128), (128, 32), (80, 80)])
def test_k4_head_dims(mbci, emu, K, L):
    inp = gen.make_chain_inputs(K + 3 * L, "bf16", 3, 256, 512, K, L, 1)
    check4(mbci, inp, 1.0 / math.sqrt(K))


@pytest.mark.parametrize("M,N,K,L", [(300, 333, 48, 40), (129, 1000, 72, 56), (1, 1, 16, 16), (384, 130, 8, 8),
                                     (640, 257, 64, 64)])
def test_k4_ragged(mbci, emu, M, N, K, L):
    inp = gen.make_chain_inputs(M + N, "f16", 2, M, N, K, L, 1)
    check4(mbci, inp, 1.0 / math.sqrt(K))


def test_k4_key_padding_mixed(mbci, emu):
    b = 9
    inp = gen.make_chain_inputs(5, "f16", b, 256, 512, 64, 64, 1, sigmas=(3.0, 3.0, 1.0))
    vl = np.array([512, 1, 0, 130, 128, 257, 0, 511, 2], dtype=np.int32)
    E, _ = check4(mbci, inp, 0.125, valid_len=vl)
    got = e_f64(E, "f16")
    D = gen.bits_to_f64_numpy(inp.D, "f16")
    assert np.array_equal(got[1], np.broadcast_to(D[1, 0], got[1].shape))   # one key: E = D[0,:]
    assert np.all(got[2] == 0.0) and np.all(got[6] == 0.0)                  # no key: E = 0


def test_k4_rescale_path_rising_scores(mbci, emu):
    base = gen.make_chain_inputs(9, "bf16", 2, 256, 1024, 64, 64, 1)
    A = gen.bits_to_f64_numpy(base.A, "bf16")
    B = gen.bits_to_f64_numpy(base.B, "bf16")
    A[:, :, -1] = 1.0

    def bits(x):
        return gen._f64_to_storage(x.ravel(), "bf16").reshape(x.shape)

    for gamma in (0.03125, 0.25):
        B[:, :, -1] = gamma * np.arange(1024)[None, :]
        inp = gen.ChainInputs(bits(A), bits(B), base.D, None, "bf16", 2, 256, 1024, 64, 64, 1)
        check4(mbci, inp, 1.0)


def test_k4_negative_and_zero_scale(mbci, emu):
    inp = gen.make_chain_inputs(12, "bf16", 2, 256, 384, 64, 64, 1)
    check4(mbci, inp, -0.125)
    check4(mbci, inp, 0.0)


def test_k4_rows_sum_to_one(mbci, emu):
    inp = gen.make_chain_inputs(11, "f16", 4, 256, 384, 64, 64, 1, sigmas=(2.0, 2.0, 1.0))
    inp.D = np.ascontiguousarray(np.full(inp.D.shape, 0x3C00, dtype=np.uint16))
    E, _ = run_chain(mbci, inp, "softmax", 0.125, plan=k4_plan(mbci, 64))
    assert np.max(np.abs(e_f64(E, "f16") - 1.0)) <= 2 * 2.0 ** -11 + 1e-6


@pytest.mark.parametrize("stages", [3, 4, 5])   # 5 stages leave room for one Q-pair buffer only
def test_k4_many_units_per_cta(mbci, emu, stages):
    """600 pair units on <= 148 CTAs: every Q buffer, the K/V ring and o_free cycle many times;
    key lengths vary per β so CTAs interleave units of 0..3 tiles."""
    b, M, N = 600, 256, 384
    inp = gen.make_chain_inputs(21, "f16", b, M, N, 64, 64, 1, valid_len_range=(0, N))
    rows = np.stack([np.arange(b), (np.arange(b) * 37) % M], axis=1).astype(np.int64)
    check4(mbci, inp, 0.125, valid_len=inp.valid_len, stages=stages, rows=rows)


def test_k4_wide_head_two_stages(mbci, emu):
    """TL > 64 keeps two S buffers (NSB = 2), whose K/V release needs only two ring stages."""
    inp = gen.make_chain_inputs(23, "bf16", 300, 256, 384, 128, 128, 1)
    rows = np.stack([np.arange(300), (np.arange(300) * 53) % 256], axis=1).astype(np.int64)
    check4(mbci, inp, 1.0 / math.sqrt(128), stages=2, rows=rows)


@pytest.mark.parametrize("batch,M,N", [(156, 512, 512), (96, 512, 512), (150, 256, 1024), (300, 300, 700),
                                     (4, 200, 250)])
@pytest.mark.parametrize("halves", ["on", "off"])
def test_k4_half_items(mbci, emu, batch, M, N, halves, monkeypatch):
    """A last round of <= 74 pair units runs as half items: one 128-row Q tile per CTA whose two
    slots split the key tiles, merged by log-sum-exp in the epilogue.  Sampled rows plus every
    row of the last pair units (the half items), both settings, and run-to-run determinism."""
    if halves == "off":
        monkeypatch.setenv("MBCI_T4_NO_HALF", "1")
    inp = gen.make_chain_inputs(31 + batch, "f16", batch, M, N, 64, 64, 1, sigmas=(2.0, 2.0, 1.0))
    last = batch - 1
    rows = np.stack([np.arange(batch), (np.arange(batch) * 101) % M], axis=1).astype(np.int64)
    rows = np.concatenate([rows, np.stack([np.full(M, last), np.arange(M)], axis=1)]).astype(np.int64)
    E1, ch = check4(mbci, inp, 0.125, rows=rows, stages=4)   # halves need a 4-deep ring at d = 64
    E2, _ = run_chain(mbci, inp, "softmax", 0.125, plan=k4_plan(mbci, 64, stages=4))
    assert torch.equal(E1.view(torch.int16), E2.view(torch.int16))


@pytest.mark.parametrize("dtype,b_layout,K,L", [("bf16", 0, 64, 64), ("bf16", 1, 48, 40), ("f16", 0, 32, 64)])
def test_k4_half_items_layouts(mbci, dtype, b_layout, K, L):
    """Half items with B stored [K, N] (MN-major K tiles), bf16, and head dims below 64."""
    batch, M, N = 150, 256, 512
    inp = gen.make_chain_inputs(77 + K, dtype, batch, M, N, K, L, b_layout)
    rows = np.concatenate([np.stack([np.full(M, batch - 1), np.arange(M)], axis=1),
                           np.stack([np.arange(batch), (np.arange(batch) * 53) % M], axis=1)]).astype(np.int64)
    check4(mbci, inp, 1.0 / math.sqrt(K), rows=rows, stages=4)


def test_k4_deterministic(mbci, emu):
    inp = gen.make_chain_inputs(17, "f16", 16, 512, 512, 64, 64, 1)
    E1, _ = run_chain(mbci, inp, "softmax", 0.125, plan=k4_plan(mbci, 64))
    E2, _ = run_chain(mbci, inp, "softmax", 0.125, plan=k4_plan(mbci, 64))
    assert torch.equal(E1.view(torch.int16), E2.view(torch.int16))


def test_k4_strided_operands(mbci):
    b, M, N, K, L = 3, 200, 320, 64, 48
    inp = gen.make_chain_inputs(16, "f16", b, M, N, K, L, 1)

    def pad(x, ld, bs):
        out = np.zeros(b * bs, dtype=np.uint16)
        rows, cols = x.shape[1], x.shape[2]
        v = out.reshape(b, bs)
        for i in range(b):
            v[i, :rows * ld].reshape(rows, ld)[:, :cols] = x[i]
        return out

    ldA, bsA, ldB, bsB, ldD, bsD, ldE, bsE = 72, 72 * 200 + 64, 80, 80 * 320, 56, 56 * 320 + 8, 64, 64 * 200 + 16
    A, B, D = (to_dev(pad(inp.A, ldA, bsA), "f16"), to_dev(pad(inp.B, ldB, bsB), "f16"),
               to_dev(pad(inp.D, ldD, bsD), "f16"))
    E = torch.full((b * bsE,), float("nan"), dtype=torch.float16, device="cuda")
    ch = mbci.Chain(b, M, N, K, L, "f16", "softmax", 0.125, b_layout=1, plan=k4_plan(mbci, L),
                    strides=dict(ld_a=ldA, bs_a=bsA, ld_b=ldB, bs_b=bsB, ld_d=ldD, bs_d=bsD, ld_e=ldE, bs_e=bsE))
    assert ch.plan().kernel == _KERN["k"]
    ch.run(A, B, D, E)
    torch.cuda.synchronize()
    Ef = E.cpu().float().numpy().astype(np.float64).reshape(b, bsE)
    got = np.stack([Ef[i, :M * ldE].reshape(M, ldE)[:, :L] for i in range(b)])
    assert np.all(np.isnan(Ef[0, M * ldE:]))
    assert np.all(np.isnan(Ef[0, :ldE * M].reshape(M, ldE)[:, L:]))
    assert oracle.row_max_error(got, oracle.chain(inp, "softmax", 0.125)) <= BUDGET["f16"]


# ------------------------------------------------------------------ NONE / SCALE on kernel 4
@pytest.mark.parametrize("dtype,K", [("f16", 16), ("f16", 64), ("bf16", 32), ("bf16", 128), ("f16", 128)])
@pytest.mark.parametrize("b_layout", [0, 1])
def test_k4_plain_chain_integer_bitwise(mbci, dtype, K, b_layout):
    """Integers in [-2, 2]: every product and fp32 partial sum is exact, so E must equal
    RN-even(oracle E) bit for bit (SURVEY §8(c) pin), for NONE and SCALE (0.5)."""
    inp = gen.make_chain_inputs(200 + K, dtype, 3, 384, 640, K, K, b_layout, kind="int")
    for op, sc in (("none", 1.0), ("scale", 0.5)):
        E, ch = run_chain(mbci, inp, op, sc, plan=k4_plan(mbci, K, K=K))
        assert ch.plan().kernel == _KERN["k"], ch.describe()
        ref = oracle.chain(inp, op, sc)
        assert np.array_equal(e_bits(E), rn_bits(ref, dtype)), ch.describe()


@pytest.mark.parametrize("M,N,K,L", [(300, 333, 48, 40), (129, 1000, 72, 56), (1, 1, 16, 16)])
def test_k4_plain_chain_ragged(mbci, M, N, K, L):
    sig = (1.0, 1.0 / math.sqrt(K), 1.0 / math.sqrt(N))
    inp = gen.make_chain_inputs(M + N + 7, "bf16", 2, M, N, K, L, 1, sigmas=sig)
    for op, sc in (("none", 1.0), ("scale", -0.75)):
        E, ch = run_chain(mbci, inp, op, sc, plan=k4_plan(mbci, L, K=K))
        err = oracle.row_max_error(e_f64(E, "bf16"), oracle.chain(inp, op, sc))
        assert err <= BUDGET["bf16"], (op, err, ch.describe())


@pytest.mark.parametrize("op", ["none", "scale"])
def test_k4_plain_chain_half_items(mbci, op):
    """NONE / SCALE through half items: the two slots' partial products are summed (no
    normalisation).  156 x 512 rows -> 312 pair units -> the last 16 run as half items."""
    b, M, N, K = 156, 512, 512, 64
    inp = gen.make_chain_inputs(5, "bf16", b, M, N, K, K, 1, sigmas=(1.0, 1.0 / math.sqrt(K), 1.0 / math.sqrt(N)))
    E, ch = run_chain(mbci, inp, op, 0.5 if op == "scale" else 1.0, plan=k4_plan(mbci, K, stages=4))
    rows = np.concatenate([np.stack([np.full(M, b - 1), np.arange(M)], axis=1),
                           np.stack([np.arange(b), (np.arange(b) * 37) % M], axis=1)]).astype(np.int64)
    ref = oracle.chain(inp, op, 0.5 if op == "scale" else 1.0, rows=rows)
    err = oracle.row_max_error(e_f64(E, "bf16")[rows[:, 0], rows[:, 1]], ref)
    assert err <= BUDGET["bf16"], (err, ch.describe())


def test_k4_plain_chain_C4_shape_sampled(mbci):
    b, M, N, K = 64, 2048, 2048, 64
    inp = gen.make_chain_inputs(0, "bf16", b, M, N, K, K, 0, sigmas=(1.0, 1.0 / math.sqrt(K), 1.0 / math.sqrt(N)))
    E, ch = run_chain(mbci, inp, "none", 1.0, plan=k4_plan(mbci, K))
    rows = np.stack([np.arange(b), (np.arange(b) * 389) % M], axis=1).astype(np.int64)
    ref = oracle.chain(inp, "none", 1.0, rows=rows)
    err = oracle.row_max_error(e_f64(E, "bf16")[rows[:, 0], rows[:, 1]], ref)
    assert err <= BUDGET["bf16"], (err, ch.describe())
