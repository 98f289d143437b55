"""Parity of kernel 7 (chain_tf32.cuh: fp32 on tcgen05 tensor cores, kind::tf32 with 3xTF32
compensation) with the fp64 oracle, through the C ABI.  Tolerance: BASELINE.json north_star's
1e-5 (row-max-normalised, R10) on every case; integer chains must match RN(oracle) bit
for bit (every TF32 split is exact: lo = 0, and every fp32 partial sum is an exact integer).

Covers the C1 config, both B layouts, every op, ragged M / N / K / L up to 128 (the wide 32-key-tile
variant for K or L > 64; K not a multiple of 8, L not of 16, N not of 64), key padding (0, 1, partial and full lengths), the online-rescale path, negative
and zero scale, unaligned strides (kernel 7 reads global memory with scalar loads), agreement with
the CUDA-core kernel, run-to-run determinism, and that the default fp32 plan is kernel 7.
"""
import math

import numpy as np
import pytest
import torch

import mbci_inputs as gen
import oracle
from gpu_helpers import e_bits, e_f64, rn_bits, run_chain, to_dev

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def mbci():
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    from paper_2506_22169_b200 import mbci as m
    return m


def k7(mbci):
    p = mbci.mbci_plan_t()
    p.kernel = 7
    return p


def check7(mbci, inp, op, scale, valid_len=None):
    E, ch = run_chain(mbci, inp, op, scale, valid_len, plan=k7(mbci))
    assert ch.plan().kernel == 7, ch.describe()
    got = e_f64(E, "f32")
    ref = oracle.chain(inp, op, scale, valid_len=valid_len)
    assert np.all(np.isfinite(got))
    err = oracle.row_max_error(got, ref)
    assert err <= TOL, (err, ch.describe())
    return E, err


def test_default_fp32_plan_is_kernel7(mbci):
    inp = gen.make_chain_inputs(0, "f32", 1, 128, 128, 16, 16, 0)
    E, ch = run_chain(mbci, inp, "none", 1.0)
    assert ch.plan().kernel == 7 and "tf32x3" in ch.describe()
    assert oracle.row_max_error(e_f64(E, "f32"), oracle.chain(inp, "none", 1.0)) <= TOL


@pytest.mark.parametrize("K", [8, 16, 40, 64, 128])
@pytest.mark.parametrize("b_layout", [0, 1])
def test_integer_chain_bitwise(mbci, K, b_layout):
    inp = gen.make_chain_inputs(300 + K, "f32", 3, 200, 300, K, 48, b_layout, kind="int")
    for op, sc in (("none", 1.0), ("scale", 0.5)):
        E, ch = run_chain(mbci, inp, op, sc, plan=k7(mbci))
        assert np.array_equal(e_bits(E), rn_bits(oracle.chain(inp, op, sc), "f32")), ch.describe()


@pytest.mark.parametrize("op,scale", [("none", 1.0), ("scale", -0.75), ("softmax", 0.25), ("softmax", None)])
@pytest.mark.parametrize("b_layout", [0, 1])
def test_ops_and_layouts(mbci, op, scale, b_layout):
    inp = gen.make_chain_inputs(7, "f32", 4, 256, 320, 32, 64, b_layout)
    check7(mbci, inp, op, 1.0 / math.sqrt(32) if scale is None else scale)


@pytest.mark.parametrize("M,N,K,L", [(1, 1, 1, 1), (129, 65, 9, 17), (300, 333, 20, 40), (100, 130, 24, 20),
                                     (64, 1000, 64, 64), (257, 64, 63, 33), (200, 300, 128, 128), (130, 77, 96, 40),
                                     (64, 200, 24, 120)])
def test_ragged_shapes(mbci, M, N, K, L):
    inp = gen.make_chain_inputs(M + N + K, "f32", 2, M, N, K, L, 1)
    check7(mbci, inp, "softmax", 1.0 / math.sqrt(K))
    check7(mbci, inp, "none", 1.0)


def test_key_padding(mbci):
    inp = gen.make_chain_inputs(5, "f32", 6, 128, 300, 32, 32, 1, sigmas=(2.0, 2.0, 1.0))
    vl = np.array([300, 1, 0, 65, 64, 299], dtype=np.int32)
    E, _ = check7(mbci, inp, "softmax", 0.25, valid_len=vl)
    got = e_f64(E, "f32")
    D = gen.bits_to_f64_numpy(inp.D, "f32")
    # one key: E = D[0, :] up to the tensor core's recombination of D_hi + D_lo (not exact in its
    # accumulator: 3xTF32 carries ~2^-22 relative)
    assert np.max(np.abs(got[1] - D[1, 0][None, :])) <= 1e-6 * np.max(np.abs(D[1, 0]))
    assert np.all(got[2] == 0.0)                                             # no key: E = 0


def test_rescale_path_rising_scores(mbci):
    """Key scores rising along n force the online rescale at every tile.  Scale 0.05 keeps
    |scale * S| <= ~20: fp32 scores near 256 carry an ulp of 3e-5 that the exponential turns into a
    relative error above 1e-5 on any fp32 path (an input-range limit, not a kernel one)."""
    base = gen.make_chain_inputs(9, "f32", 2, 128, 512, 16, 16, 1)
    A = gen.bits_to_f64_numpy(base.A, "f32")
    B = gen.bits_to_f64_numpy(base.B, "f32")
    A[:, :, -1] = 1.0
    for gamma in (0.01, 0.5):
        B[:, :, -1] = gamma * np.arange(512)[None, :]
        bits = lambda x: gen._f64_to_storage(x.ravel(), "f32").reshape(x.shape)
        inp = gen.ChainInputs(bits(A), bits(B), base.D, None, "f32", 2, 128, 512, 16, 16, 1)
        check7(mbci, inp, "softmax", 0.05)


def test_negative_and_zero_scale(mbci):
    inp = gen.make_chain_inputs(12, "f32", 2, 128, 200, 16, 16, 1)
    check7(mbci, inp, "softmax", -0.5)
    check7(mbci, inp, "softmax", 0.0)


def test_unaligned_strides(mbci):
    """Row strides that are not 16-byte multiples (illegal for TMA) stay on kernel 7."""
    b, M, N, K, L = 2, 130, 150, 13, 11
    inp = gen.make_chain_inputs(16, "f32", b, M, N, K, L, 1)

    def pad(x, ld, bs):
        out = np.zeros(b * bs, dtype=np.uint32)
        rows, cols = x.shape[1], x.shape[2]
        v = out.reshape(b, bs)
        for i in range(b):
            v[i, :rows * ld].reshape(rows, ld)[:, :cols] = x[i]
        return out

    ldA, bsA, ldB, bsB, ldD, bsD, ldE, bsE = 15, 15 * 130 + 3, 17, 17 * 150, 13, 13 * 150 + 1, 12, 12 * 130 + 5
    A, B, D = to_dev(pad(inp.A, ldA, bsA), "f32"), to_dev(pad(inp.B, ldB, bsB), "f32"), to_dev(pad(inp.D, ldD, bsD), "f32")
    E = torch.full((b * bsE,), float("nan"), dtype=torch.float32, device="cuda")
    ch = mbci.Chain(b, M, N, K, L, "f32", "softmax", 0.3, b_layout=1, plan=k7(mbci),
                    strides=dict(ld_a=ldA, bs_a=bsA, ld_b=ldB, bs_b=bsB, ld_d=ldD, bs_d=bsD, ld_e=ldE, bs_e=bsE))
    assert ch.plan().kernel == 7
    ch.run(A, B, D, E)
    torch.cuda.synchronize()
    Ef = E.cpu().numpy().astype(np.float64).reshape(b, bsE)
    got = np.stack([Ef[i, :M * ldE].reshape(M, ldE)[:, :L] for i in range(b)])
    assert np.all(np.isnan(Ef[0, :ldE * M].reshape(M, ldE)[:, L:]))
    assert oracle.row_max_error(got, oracle.chain(inp, "softmax", 0.3)) <= TOL


def test_agrees_with_cuda_cores_and_is_deterministic(mbci):
    inp = gen.make_chain_inputs(21, "f32", 3, 256, 384, 64, 64, 0)
    E1, _ = run_chain(mbci, inp, "softmax", 0.125, plan=k7(mbci))
    E2, _ = run_chain(mbci, inp, "softmax", 0.125, plan=k7(mbci))
    assert torch.equal(E1, E2)
    p1 = mbci.mbci_plan_t()
    p1.kernel = 1
    E3, _ = run_chain(mbci, inp, "softmax", 0.125, plan=p1)
    ref = oracle.chain(inp, "softmax", 0.125)
    assert oracle.row_max_error(e_f64(E1, "f32"), ref) <= TOL
    assert oracle.row_max_error(e_f64(E3, "f32"), ref) <= TOL
