"""Parity of the CUDA path (through the C ABI) with the fp64 CPU oracle.

Tolerances (BASELINE.json north star): fp16/bf16 row-max-normalised error <= 2e-2, fp32
<= 1e-5.  Exact cases (integer inputs whose products and sums are exact in the 16-bit
type and fp32) must match RN-even(oracle) bit for bit.  A second, tighter bound per
dtype (DESIGN.md §4 error budget) flags a kernel bug that still fits the contract.
"""
import math

import numpy as np
import pytest
import torch

import mbci_inputs as gen
import oracle
from gpu_helpers import e_bits, e_f64, rn_bits, run_chain, to_dev

pytestmark = pytest.mark.gpu

TOL = {"f16": 2e-2, "bf16": 2e-2, "f32": 1e-5}
BUDGET = {"f16": 4e-3, "bf16": 1.5e-2, "f32": 1e-5}   # ~4x the emulated worst case


@pytest.fixture(scope="module")
def mbci():
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    from paper_2506_22169_b200 import mbci as m
    return m


def check(mbci, inp, op, scale, valid_len=None, plan=None, budget=True):
    E, ch = run_chain(mbci, inp, op, scale, valid_len, plan)
    got = e_f64(E, inp.dtype)
    ref = oracle.chain(inp, op, scale, valid_len=valid_len)
    err = oracle.row_max_error(got, ref)
    assert np.all(np.isfinite(got)), "non-finite output"
    assert err <= TOL[inp.dtype], (err, ch.describe())
    if budget:
        assert err <= BUDGET[inp.dtype], (err, ch.describe())
    return err, ch


# ------------------------------------------------------------------ exact (bitwise) cases
@pytest.mark.parametrize("dtype,K", [("f16", 16), ("f16", 64), ("f16", 128), ("bf16", 16), ("bf16", 32),
                                     ("bf16", 64)])
@pytest.mark.parametrize("b_layout", [0, 1])
def test_integer_chain_bitwise(mbci, dtype, K, b_layout):
    """Integers in [-2,2]: |C| <= 4K is exact in the 16-bit type, E's fp32 sums are exact,
    so E must equal RN-even(oracle E) bit for bit (SURVEY §8(c) pin)."""
    inp = gen.make_chain_inputs(100 + K, dtype, 2, 384, 640, K, K, b_layout, kind="int")
    for op, sc in (("none", 1.0), ("scale", 0.5)):
        E, ch = run_chain(mbci, inp, op, sc)
        ref = oracle.chain(inp, op, sc)
        assert np.array_equal(e_bits(E), rn_bits(ref, dtype)), ch.describe()


def test_identity_D_exposes_scores(mbci):
    """D = I (L = N = 128): E = A·B exactly for integer inputs."""
    inp = gen.make_chain_inputs(7, "f16", 3, 256, 128, 64, 128, 1, kind="int")
    eye = np.broadcast_to(np.eye(128, dtype=np.float16).view(np.uint16), (3, 128, 128))
    inp.D = np.ascontiguousarray(eye)
    E, _ = run_chain(mbci, inp, "none", 1.0)
    ref = oracle.chain(inp, "none")
    assert np.array_equal(e_bits(E), rn_bits(ref, "f16"))


# ------------------------------------------------------------------ softmax / scale / none
@pytest.mark.parametrize("dtype,b_layout", [("f16", 1), ("bf16", 1), ("f16", 0), ("bf16", 0)])
def test_bert_base_head_slice(mbci, dtype, b_layout):
    inp = gen.make_chain_inputs(1, dtype, 8, 512, 512, 64, 64, b_layout)
    check(mbci, inp, "softmax", 0.125)


@pytest.mark.parametrize("op", ["none", "scale", "softmax"])
@pytest.mark.parametrize("K,L", [(16, 16), (32, 32), (64, 64), (128, 128), (80, 80), (64, 128), (128, 32)])
def test_ops_and_head_dims(mbci, op, K, L):
    sig = (1.0, 1.0 / math.sqrt(K), 1.0 / math.sqrt(512)) if op != "softmax" else (1.0, 1.0, 1.0)
    inp = gen.make_chain_inputs(K * 7 + L, "bf16", 3, 256, 512, K, L, 1, sigmas=sig)
    check(mbci, inp, op, 0.7 if op == "scale" else 1.0 / math.sqrt(K))


@pytest.mark.parametrize("M,N,K,L", [(300, 333, 64, 40), (1, 1, 16, 16), (129, 65, 48, 24), (77, 1000, 72, 56),
                                     (128, 130, 8, 8)])
@pytest.mark.parametrize("b_layout", [0, 1])
def test_ragged_shapes(mbci, M, N, K, L, b_layout):
    """Shapes that are not multiples of the tiles.  Packed B[K,N] with N % 8 != 0 has a row
    stride that is not a 16-B multiple (not TMA-legal): the selector must fall back to the
    CUDA-core kernel, which is checked against the oracle like every other path."""
    inp = gen.make_chain_inputs(M + N, "f16", 2, M, N, K, L, b_layout)
    _, ch = check(mbci, inp, "softmax", 1.0 / math.sqrt(K))
    check(mbci, inp, "none", 1.0, budget=False)
    if b_layout == 0 and N % 8:
        assert ch.plan().kernel == 1, ch.describe()
    elif K % 8 == 0 and L % 8 == 0 and not (b_layout == 1 and K % 8):
        assert ch.plan().kernel != 1, ch.describe()


def test_key_padding_mask(mbci):
    inp = gen.make_chain_inputs(5, "f16", 6, 256, 512, 64, 64, 1, sigmas=(3.0, 3.0, 1.0))
    vl = np.array([512, 1, 0, 130, 128, 257], dtype=np.int32)
    err, _ = check(mbci, inp, "softmax", 0.125, valid_len=vl)
    E, _ = run_chain(mbci, inp, "softmax", 0.125, valid_len=vl)
    got = e_f64(E, "f16")
    D = gen.bits_to_f64_numpy(inp.D, "f16")
    assert np.array_equal(got[1], np.broadcast_to(D[1, 0], got[1].shape))  # one key: E = D[0,:]
    assert np.all(got[2] == 0.0)                                               # no key: E = 0


def test_rescale_path_rising_scores(mbci):
    """Key scores rise with n (extra K column: A[:,K-1] = 1, B[n,K-1] = gamma*n) so every
    row's running max grows on every n-tile: exercises the lazy O rescale."""
    base = gen.make_chain_inputs(9, "bf16", 2, 256, 1024, 64, 64, 1)
    A = gen.bits_to_f64_numpy(base.A, "bf16")
    B = gen.bits_to_f64_numpy(base.B, "bf16")
    A[:, :, -1] = 1.0
    B[:, :, -1] = 0.03125 * np.arange(1024)[None, :]    # +4 per 128-key tile after scaling by 1
    def bits(x):
        return gen._f64_to_storage(x.ravel(), "bf16").reshape(x.shape)
    inp = gen.ChainInputs(bits(A), bits(B), base.D, None, "bf16", 2, 256, 1024, 64, 64, 1)
    check(mbci, inp, "softmax", 1.0)
    B[:, :, -1] = 0.25 * np.arange(1024)[None, :]       # large jumps: always past the threshold
    inp.B = bits(B)
    check(mbci, inp, "softmax", 1.0)


def test_softmax_rows_sum_to_one(mbci):
    inp = gen.make_chain_inputs(11, "f16", 4, 256, 384, 64, 64, 1, sigmas=(2.0, 2.0, 1.0))
    inp.D = np.ascontiguousarray(np.full(inp.D.shape, 0x3C00, dtype=np.uint16))   # D = ones (fp16 1.0)
    E, _ = run_chain(mbci, inp, "softmax", 0.125)
    assert np.max(np.abs(e_f64(E, "f16") - 1.0)) <= 2 * 2.0 ** -11 + 1e-6


def test_negative_and_zero_scale(mbci):
    inp = gen.make_chain_inputs(12, "bf16", 2, 128, 256, 64, 64, 1)
    check(mbci, inp, "softmax", -0.125)
    check(mbci, inp, "softmax", 0.0)


# ------------------------------------------------------------------ degenerate shapes
def test_zero_N_writes_zeros(mbci):
    inp = gen.make_chain_inputs(13, "f16", 2, 130, 0, 64, 64, 1)
    for op in ("none", "softmax"):
        E, _ = run_chain(mbci, inp, op, 0.125)
        assert torch.all(E == 0)


def test_zero_K(mbci):
    inp = gen.make_chain_inputs(14, "bf16", 2, 200, 300, 0, 64, 1)
    E, _ = run_chain(mbci, inp, "none", 1.0)
    assert torch.all(E == 0)
    check(mbci, inp, "softmax", 0.125)   # uniform mean of the D rows


def test_zero_batch_M_L_launch_nothing(mbci):
    for (b, M, L) in ((0, 64, 64), (2, 0, 64), (2, 64, 0)):
        ch = mbci.Chain(b, M, 128, 64, L, "f16", "softmax", 0.125)
        assert ch.launches_per_run() == 0
        E = torch.empty(max(b, 1), max(M, 1), max(L, 1), dtype=torch.float16, device="cuda")
        x = torch.empty(16, dtype=torch.float16, device="cuda")
        ch.run(x, x, x, E)


def test_misaligned_pointer_rejected(mbci):
    inp = gen.make_chain_inputs(15, "f16", 1, 128, 128, 64, 64, 1)
    ch = mbci.Chain(1, 128, 128, 64, 64, "f16", "softmax", 0.125)
    A = to_dev(np.concatenate([inp.A.ravel(), np.zeros(8, np.uint16)]), "f16")
    B, D = to_dev(inp.B, "f16"), to_dev(inp.D, "f16")
    E = torch.empty(1, 128, 64, dtype=torch.float16, device="cuda")
    with pytest.raises(mbci.MbciError) as ei:
        ch.run_ptr(A.data_ptr() + 2, B.data_ptr(), D.data_ptr(), E.data_ptr(), 0,
                   torch.cuda.current_stream().cuda_stream)
    assert ei.value.status == mbci.MBCI_ERR_UNSUPPORTED


# ------------------------------------------------------------------ strides
@pytest.mark.parametrize("kernel", [0, 4, 5])
def test_strided_operands(mbci, kernel):
    """Rows padded (ld > inner) and batch strides with gaps, 16-B multiples (TMA-legal),
    on every tensor-core kernel family."""
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
    pl = mbci.mbci_plan_t()
    pl.kernel, pl.BN, pl.TL, pl.stages = kernel, 128, 48, (2 if kernel == 0 else 4)
    ch = mbci.Chain(b, M, N, K, L, "f16", "softmax", 0.125, b_layout=1, plan=pl,
                    strides=dict(ld_a=ldA, bs_a=bsA, ld_b=ldB, bs_b=bsB, ld_d=ldD, bs_d=bsD, ld_e=ldE, bs_e=bsE))
    assert ch.plan().kernel == kernel
    ch.run(A, B, D, E)
    torch.cuda.synchronize()
    Ef = E.cpu().float().numpy().astype(np.float64).reshape(b, bsE)
    got = np.stack([Ef[i, :M * ldE].reshape(M, ldE)[:, :L] for i in range(b)])
    assert np.all(np.isnan(Ef[0, M * ldE:]))           # gaps between batches untouched
    assert np.all(np.isnan(Ef[0, :ldE * M].reshape(M, ldE)[:, L:]))   # row padding untouched
    err = oracle.row_max_error(got, oracle.chain(inp, "softmax", 0.125))
    assert err <= BUDGET["f16"]


# ------------------------------------------------------------------ fp32 + CUDA-core path
def test_fp32_chain_C1(mbci):
    """BASELINE config 0: fp32, batch 1, M=N=128, K=L=16, no inter-op, 1e-5 — on the default plan
    (kernel 7, tcgen05 3xTF32) and on the CUDA-core fallback (kernel 1)."""
    inp = gen.make_chain_inputs(0, "f32", 1, 128, 128, 16, 16, 0)
    err, ch = check(mbci, inp, "none", 1.0)
    assert ch.plan().kernel == 7
    k1 = mbci.mbci_plan_t()
    k1.kernel = 1
    err, ch = check(mbci, inp, "none", 1.0, plan=k1)
    assert ch.plan().kernel == 1
    inp2 = gen.make_chain_inputs(1, "f32", 2, 100, 130, 24, 20, 1)
    for plan in (None, k1):
        check(mbci, inp2, "softmax", 0.2, plan=plan)


def test_unaligned_16bit_uses_cuda_cores(mbci):
    inp = gen.make_chain_inputs(2, "bf16", 2, 3, 5, 3, 3, 0)
    err, ch = check(mbci, inp, "softmax", 0.5)
    assert ch.plan().kernel == 1


# ------------------------------------------------------------------ plans, determinism, e2e
def test_every_plan_agrees_and_is_deterministic(mbci):
    inp = gen.make_chain_inputs(17, "f16", 4, 256, 512, 64, 64, 1)
    ref = oracle.chain(inp, "softmax", 0.125)
    st, plans = mbci.plan_enumerate(mbci.make_desc(4, 256, 512, 64, 64, "f16", "softmax", 0.125))
    assert st == 0 and len(plans) >= 6
    for p in plans:
        E1, ch = run_chain(mbci, inp, "softmax", 0.125, plan=p)
        E2, _ = run_chain(mbci, inp, "softmax", 0.125, plan=p)
        assert torch.equal(E1.view(torch.int16), E2.view(torch.int16)), ch.describe()
        assert oracle.row_max_error(e_f64(E1, "f16"), ref) <= BUDGET["f16"], ch.describe()


def test_tune_mode_picks_a_legal_plan(mbci):
    inp = gen.make_chain_inputs(18, "f16", 8, 512, 512, 64, 64, 1)
    E, ch = run_chain(mbci, inp, "softmax", 0.125, tune=1)
    assert oracle.row_max_error(e_f64(E, "f16"), oracle.chain(inp, "softmax", 0.125)) <= BUDGET["f16"]


def test_run_host_matches_device_run(mbci):
    inp = gen.make_chain_inputs(19, "bf16", 4, 256, 256, 64, 64, 1, valid_len_range=(1, 256))
    Ed, ch = run_chain(mbci, inp, "softmax", 0.125, valid_len=inp.valid_len)
    Eh = torch.empty(4, 256, 64, dtype=torch.bfloat16).pin_memory()
    pin = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).pin_memory()
    ch.run_host(pin(inp.A), pin(inp.B), pin(inp.D), Eh, torch.from_numpy(inp.valid_len).pin_memory())
    assert torch.equal(Eh.view(torch.int16), Ed.cpu().view(torch.int16))


# ------------------------------------------------------------------ full-size configs, sampled
def _sample_rows(batch, M, n, seed):
    rng = np.random.default_rng(seed)
    rows = np.stack([rng.integers(0, batch, n), rng.integers(0, M, n)], axis=1)
    rows[:4] = [[0, 0], [batch - 1, M - 1], [0, M - 1], [batch - 1, 0]]
    return rows.astype(np.int64)


FULL_CONFIGS = [
    ("C2", "f16", 96, 512, 512, 64, 64),
    ("C3", "bf16", 128, 1024, 1024, 64, 64),
    ("C4-16", "bf16", 64, 2048, 2048, 16, 16),
    ("C4-32", "bf16", 64, 2048, 2048, 32, 32),
    ("C4-64", "bf16", 64, 2048, 2048, 64, 64),
    ("C4-128", "bf16", 64, 2048, 2048, 128, 128),
    ("C5", "bf16", 512, 4096, 4096, 128, 128),
    ("C6", "f16", 96, 256, 256, 64, 64),
]


@pytest.mark.parametrize("cfg", FULL_CONFIGS, ids=[c[0] for c in FULL_CONFIGS])
def test_full_size_configs_sampled(mbci, cfg):
    """BASELINE.json configs at full size, default plan (the one bench.py times): 256 sampled
    (β, m) rows, including the first and last β and row, each computed by the oracle alone."""
    name, dtype, b, M, N, K, L = cfg
    op = "none" if name.startswith("C4") else "softmax"
    sig = (1.0, 1.0 / math.sqrt(K), 1.0 / math.sqrt(N)) if op == "none" else (1.0, 1.0, 1.0)
    inp = gen.make_chain_inputs(0, dtype, b, M, N, K, L, 1 if op == "softmax" else 0, sigmas=sig)
    sc = 1.0 / math.sqrt(K) if op == "softmax" else 1.0
    E, ch = run_chain(mbci, inp, op, sc)
    assert ch.plan().kernel != 1, ch.describe()
    rows = _sample_rows(b, M, 256, 1)
    ref = oracle.chain(inp, op, sc, rows=rows)
    ix = torch.from_numpy(rows).to(E.device)
    got = e_f64(E[ix[:, 0], ix[:, 1]], dtype)
    err = oracle.row_max_error(got, ref)
    assert np.all(np.isfinite(got))
    assert err <= BUDGET[dtype], (name, err, ch.describe())


def test_shard_is_bitwise_slice_of_full_run(mbci):
    """rank r of g owns β in [r·b/g, (r+1)·b/g).  With the plan pinned, a shard's E
    (inputs generated for batch_start = lo only) equals those rows of the unsharded run bit for bit."""
    from paper_2506_22169_b200 import sharding
    b, M, N, K, L = 24, 512, 512, 64, 64
    full = gen.make_chain_inputs(3, "f16", b, M, N, K, L, 1)
    E_full, ch = run_chain(mbci, full, "softmax", 0.125)
    pin = ch.plan()
    for r, g in ((1, 2), (3, 4), (7, 8)):
        lo, hi = sharding.shard_range(b, r, g)
        part = gen.make_chain_inputs(3, "f16", hi - lo, M, N, K, L, 1, batch_start=lo)
        assert np.array_equal(part.A, full.A[lo:hi]) and np.array_equal(part.D, full.D[lo:hi])
        E_part, ch2 = run_chain(mbci, part, "softmax", 0.125, plan=pin)
        assert ch2.plan().kernel == pin.kernel
        assert torch.equal(E_part.view(torch.int16), E_full[lo:hi].view(torch.int16)), (r, g, ch2.describe())
