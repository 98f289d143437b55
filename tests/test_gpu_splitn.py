"""Split-N on the GPU: the chain over disjoint key ranges through
mbci_chain_run_partial (B, D as strided views at the range's first key, the full-sequence valid_len
plus the key offset), then mbci_merge_partials — against the fp64 oracle's full chain, and each part's
row log-sum-exp against oracle.row_lse of that key range.

Tolerances: the contract's 2e-2 (row-max, R10) and the per-dtype budget of
test_gpu_parity.py; fp32 (kernels 7 / 1) 1e-5; integer NONE chains in fp32 bit for bit (every
partial and every sum is an exact integer).  The lse of a part is checked to 2e-3 absolute (the
exponentials of the row sum are ex2.approx / a degree-3 polynomial, ~1e-4 relative)."""
import math

import numpy as np
import pytest
import torch

import mbci_inputs as gen
import oracle
from gpu_helpers import TORCH_DT, e_bits, e_f64, rn_bits, to_dev
from paper_2506_22169_b200 import sharding
from split_util import local_valid, lse_combine, slice_keys

pytestmark = pytest.mark.gpu

BUDGET = {"f16": 4e-3, "bf16": 1.5e-2, "f32": 1e-5}


@pytest.fixture(scope="module")
def mbci():
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    from paper_2506_22169_b200 import mbci as m
    return m


def plan_of(mbci, kernel, inp, n_keys, op, masked):
    """The selector's best legal plan of `kernel` for this part's shape (kernels 1 / 7 need no tile
    parameters)."""
    if kernel is None:
        return None
    if kernel in (1, 7):
        p = mbci.mbci_plan_t()
        p.kernel = kernel
        return p
    d = mbci.make_desc(inp.batch, inp.M, n_keys, inp.K, inp.L, inp.dtype, op, 0.125, mask=masked,
                       b_layout=inp.b_layout)
    plans = [p for p in mbci.plan_enumerate(d)[1] if p.kernel == kernel]
    assert plans, f"kernel {kernel} has no legal plan for this part"
    return plans[0]


def run_split(mbci, inp, op, scale, parts, valid_len=None, kernel=None, align=8):
    """Returns (merged E tensor, [(n0, n1, E_part, lse_part, plan kernel)])."""
    dev = torch.device("cuda", 0)
    dt = TORCH_DT[inp.dtype]
    A, B, D = to_dev(inp.A, inp.dtype), to_dev(inp.B, inp.dtype), to_dev(inp.D, inp.dtype)
    vl = None if valid_len is None else torch.from_numpy(np.asarray(valid_len, dtype=np.int32)).to(dev)
    b, M, N, K, L = inp.batch, inp.M, inp.N, inp.K, inp.L
    E_parts = torch.full((parts, b, M, L), float("nan"), dtype=dt, device=dev)
    lse = torch.full((parts, b, M), float("nan"), dtype=torch.float32, device=dev)
    out = []
    for r in range(parts):
        n0, n1 = sharding.key_range(N, r, parts, align)
        if inp.b_layout == 1:
            Bv, sb = B[:, n0:n1, :], {"ld_b": K, "bs_b": N * K}
        else:
            Bv, sb = B[:, :, n0:n1], {"ld_b": N, "bs_b": K * N}
        Dv = D[:, n0:n1, :]
        strides = dict(sb, ld_d=L, bs_d=N * L)
        ch = mbci.Chain(b, M, n1 - n0, K, L, inp.dtype, op, scale, mask=valid_len is not None,
                        b_layout=inp.b_layout, device=0, strides=strides,
                        plan=plan_of(mbci, kernel, inp, n1 - n0, op, valid_len is not None))
        ch.run_partial(A, Bv, Dv, E_parts[r], lse[r] if op == "softmax" else None, vl, n0)
        out.append((n0, n1, E_parts[r], lse[r], ch.plan().kernel))
        torch.cuda.synchronize()
        ch.close()
    E = torch.full((b, M, L), float("nan"), dtype=dt, device=dev)
    mbci.merge_partials(E_parts, lse if op == "softmax" else None, E, op)
    torch.cuda.synchronize()
    return E, out


def check_split(mbci, inp, op, scale, parts, valid_len=None, kernel=None, expect_kernel=None):
    E, out = run_split(mbci, inp, op, scale, parts, valid_len, kernel)
    if expect_kernel is not None:
        assert all(k == expect_kernel for *_, k in out), [k for *_, k in out]
    ref = oracle.chain(inp, op, scale, valid_len=valid_len)
    got = e_f64(E, inp.dtype)
    assert np.all(np.isfinite(got))
    err = oracle.row_max_error(got, ref)
    tol = 1e-5 if inp.dtype == "f32" else 2e-2
    assert err <= tol and err <= BUDGET[inp.dtype], (err, parts, [k for *_, k in out])
    if op == "softmax":
        for n0, n1, _, lse_r, _ in out:
            sub = slice_keys(inp, n0, n1)
            ref_l = oracle.row_lse(sub, scale, local_valid(valid_len, n0, n1))
            g = lse_r.cpu().double().numpy()
            fin = np.isfinite(ref_l)
            assert np.array_equal(np.isfinite(g), fin), (n0, n1)
            assert np.all(g[~fin] == -np.inf)
            if fin.any():
                assert np.max(np.abs(g[fin] - ref_l[fin])) <= 2e-3, (n0, n1, np.max(np.abs(g[fin] - ref_l[fin])))
    return err


@pytest.mark.parametrize("parts", [1, 2, 3, 4])
@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_split_attention_default_plan(mbci, parts, dtype):
    """BERT-shaped softmax chain (kernel 5) cut into key ranges; ragged M and N."""
    inp = gen.make_chain_inputs(40 + parts, dtype, 3, 300, 700, 64, 64, 1)
    check_split(mbci, inp, "softmax", 0.125, parts, expect_kernel=5)


@pytest.mark.parametrize("parts", [2, 3])
def test_split_key_padding(mbci, parts):
    """Full-sequence valid_len with key offsets: parts past a row's valid length are fully masked
    (lse = -inf, weight 0); lengths 0 and 1 included."""
    inp = gen.make_chain_inputs(50, "f16", 6, 256, 640, 64, 64, 1)
    vl = np.array([0, 1, 100, 300, 639, 640], dtype=np.int32)
    check_split(mbci, inp, "softmax", 0.125, parts, valid_len=vl)


@pytest.mark.parametrize("kernel,L", [(4, 128), (0, 96), (0, 64)])
def test_split_other_tensor_core_kernels(mbci, kernel, L):
    inp = gen.make_chain_inputs(60 + L, "bf16", 2, 256, 512, 64, L, 1, valid_len_range=(1, 512))
    check_split(mbci, inp, "softmax", 0.125, 3, valid_len=inp.valid_len, kernel=kernel, expect_kernel=kernel)


@pytest.mark.parametrize("kernel", [7, 1])
def test_split_fp32(mbci, kernel):
    inp = gen.make_chain_inputs(70, "f32", 2, 128, 300, 32, 32, 0, valid_len_range=(0, 300))
    check_split(mbci, inp, "softmax", 1 / math.sqrt(32), 3, valid_len=inp.valid_len, kernel=kernel,
                expect_kernel=kernel)


@pytest.mark.parametrize("op", ["none", "scale", "relu", "gelu"])
def test_split_linear_ops_sum(mbci, op):
    """Every op but SOFTMAX is linear in the partial products: E = Σ_r E_r."""
    inp = gen.make_chain_inputs(80, "bf16", 2, 256, 512, 64, 64, 0, sigmas=(1.0, 0.125, 0.0625))
    check_split(mbci, inp, op, 0.5 if op != "none" else 1.0, 2)


def test_split_integer_chain_bitwise(mbci):
    """fp32 integer NONE chain: every partial and the merged sum are exact integers, so the merged
    E equals RN(oracle) bit for bit."""
    inp = gen.make_chain_inputs(90, "f32", 2, 128, 256, 16, 32, 0, kind="int")
    E, _ = run_split(mbci, inp, "none", 1.0, 3, kernel=7)
    assert np.array_equal(e_bits(E), rn_bits(oracle.chain(inp, "none", 1.0), "f32"))


@pytest.mark.parametrize("dtype", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("L", [12, 64])
@pytest.mark.parametrize("op", ["softmax", "none"])
def test_merge_kernel_against_definition(mbci, dtype, L, op):
    """mbci_merge_partials alone (vector path for L = 64, scalar for L = 12) on random partials with
    -inf entries, against the combination written out in float64 (split_util.lse_combine)."""
    rng = np.random.default_rng(L)
    R, b, M = 4, 3, 37
    parts = rng.standard_normal((R, b, M, L))
    lse = rng.standard_normal((R, b, M)) * 4
    lse[rng.random((R, b, M)) < 0.2] = -np.inf
    lse[:, 0, 0] = -np.inf   # a row with no valid key anywhere -> 0
    dt = TORCH_DT[dtype]
    Pt = torch.from_numpy(parts).to(dt).cuda()
    Lt = torch.from_numpy(lse).float().cuda()
    E = torch.full((b, M, L), float("nan"), dtype=dt, device="cuda")
    mbci.merge_partials(Pt, Lt if op == "softmax" else None, E, op)
    torch.cuda.synchronize()
    P64 = Pt.double().cpu().numpy()
    ref = lse_combine(P64, Lt.double().cpu().numpy()) if op == "softmax" else P64.sum(axis=0)
    got = E.double().cpu().numpy()
    eps = {"f32": 1e-6, "f16": 2e-3, "bf16": 1.6e-2}[dtype]
    assert np.max(np.abs(got - ref) / (np.abs(ref) + 1.0)) <= eps
    if op == "softmax":
        assert np.all(got[0, 0] == 0.0)


def test_split_errors(mbci):
    ch = mbci.Chain(1, 128, 128, 64, 64, "f16", "softmax", 0.125, device=0, causal=True)
    x = torch.zeros(1, 128, 64, dtype=torch.float16, device="cuda")
    l = torch.zeros(1, 128, dtype=torch.float32, device="cuda")
    with pytest.raises(mbci.MbciError):
        ch.run_partial(x, x, x, x, l, None, 0)   # causal: UNSUPPORTED
    ch.close()
    ch = mbci.Chain(1, 128, 128, 64, 64, "f16", "softmax", 0.125, device=0)
    with pytest.raises(mbci.MbciError):
        ch.run_partial(x, x, x, x, None, None, 0)   # SOFTMAX without lse: INVALID
    ch.close()


def test_merge_kernel_many_parts(mbci):
    """More parts than the vector path's register budget (R > 8): the scalar path takes them."""
    rng = np.random.default_rng(7)
    R, b, M, L = 11, 2, 33, 64
    parts = rng.standard_normal((R, b, M, L))
    lse = rng.standard_normal((R, b, M)) * 3
    lse[rng.random((R, b, M)) < 0.3] = -np.inf
    Pt = torch.from_numpy(parts).to(torch.float16).cuda()
    Lt = torch.from_numpy(lse).float().cuda()
    E = torch.full((b, M, L), float("nan"), dtype=torch.float16, device="cuda")
    mbci.merge_partials(Pt, Lt, E, "softmax")
    torch.cuda.synchronize()
    ref = lse_combine(Pt.double().cpu().numpy(), Lt.double().cpu().numpy())
    got = E.double().cpu().numpy()
    assert np.max(np.abs(got - ref) / (np.abs(ref) + 1.0)) <= 2e-3
