"""Pins for the CPU oracle (oracle/): each check ties the oracle to something
other than itself — a library routine (torch SDPA, numpy matmul / fp16
conversion, scipy softmax), a closed form, an invariant, exact integer
arithmetic, or a number the paper prints.  A plausible mistake in the oracle
(dropped term, wrong sign or index, transposed operand, wrong softmax axis,
mask off-by-one, missing scale) fails at least one of them.
"""
import math
import os

import numpy as np
import pytest
import scipy.special
import torch

import mbci_inputs as gen
import oracle
from oracle import model

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _f64(inp):
    """numpy (library) decode of the inputs, independent of the oracle decoder."""
    return (gen.bits_to_f64_numpy(inp.A, inp.dtype), gen.bits_to_f64_numpy(inp.B, inp.dtype),
            gen.bits_to_f64_numpy(inp.D, inp.dtype))


def _bmat(inp, B):
    """B as [batch, K, N] whatever the stored layout."""
    return B if inp.b_layout == 0 else np.swapaxes(B, 1, 2)


def _custom(dtype, A, B, D, b_layout):
    """ChainInputs from explicit float arrays (exactly representable in dtype)."""
    def bits(x):
        x = np.asarray(x, dtype=np.float64)
        if dtype == "f32":
            return x.astype(np.float32).view(np.uint32)
        if dtype == "f16":
            return x.astype(np.float16).view(np.uint16)
        return (x.astype(np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    batch, M, K = A.shape
    N, L = D.shape[1], D.shape[2]
    return gen.ChainInputs(bits(A), bits(B), bits(D), None, dtype, batch, M, N, K, L, b_layout)


# ---------------------------------------------------------------- decoders
def test_decoders_match_numpy_all_fp16_bf16_patterns():
    allbits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    for dt in ("f16", "bf16"):
        ours = oracle.decode(allbits, dt)
        ref = gen.bits_to_f64_numpy(allbits, dt)
        nan = np.isnan(ref)
        assert np.array_equal(np.isnan(ours), nan)
        assert np.array_equal(ours[~nan], ref[~nan]), dt
    rng = np.random.default_rng(0)
    f32 = rng.integers(0, 2**32, size=200000, dtype=np.uint64).astype(np.uint32)
    ours = oracle.decode(f32, "f32")
    ref = f32.view(np.float32).astype(np.float64)
    nan = np.isnan(ref)
    assert np.array_equal(ours[~nan], ref[~nan])


# ---------------------------------------------------------------- GEMMs + layouts
def test_hand_case():
    # A=[[1,2]], B=[[3],[4]], D=[[5]]  =>  C = 1*3+2*4 = 11,  E = 55
    inp = _custom("f32", np.array([[[1.0, 2.0]]]), np.array([[[3.0], [4.0]]]),
                  np.array([[[5.0]]]), 0)
    assert oracle.chain(inp, "none")[0, 0, 0] == 55.0


@pytest.mark.parametrize("b_layout", [0, 1])
@pytest.mark.parametrize("dtype", ["f32", "f16", "bf16"])
def test_brute_force_tiny_shapes_integer_exact(dtype, b_layout):
    """All (M,N,K,L) in {1,2,3}^4: E == A@(B@D) (associativity, numpy) exactly; SCALE by 0.5."""
    seed = 11
    for M in (1, 2, 3):
        for N in (1, 2, 3):
            for K in (1, 2, 3):
                for L in (1, 2, 3):
                    inp = gen.make_chain_inputs(seed, dtype, 2, M, N, K, L, b_layout, kind="int")
                    A, B, D = _f64(inp)
                    ref = A @ (_bmat(inp, B) @ D)
                    assert np.array_equal(oracle.chain(inp, "none"), ref), (M, N, K, L)
                    assert np.array_equal(oracle.chain(inp, "scale", 0.5), 0.5 * ref)
                    seed += 1


@pytest.mark.parametrize("b_layout", [0, 1])
def test_integer_chain_exact_at_medium_size(b_layout):
    inp = gen.make_chain_inputs(3, "bf16", 3, 37, 53, 16, 24, b_layout, kind="int")
    A, B, D = _f64(inp)
    assert np.array_equal(oracle.chain(inp, "none"), A @ (_bmat(inp, B) @ D))


def test_layouts_agree():
    """b_layout 1 with B stored transposed gives the same E as b_layout 0."""
    i0 = gen.make_chain_inputs(5, "f16", 2, 9, 13, 7, 5, 0)
    i1 = gen.ChainInputs(i0.A, np.ascontiguousarray(np.swapaxes(i0.B, 1, 2)), i0.D, None,
                         "f16", 2, 9, 13, 7, 5, 1)
    for op in ("none", "scale", "softmax"):
        assert np.array_equal(oracle.chain(i0, op, 0.3), oracle.chain(i1, op, 0.3))


# ---------------------------------------------------------------- softmax op
@pytest.mark.parametrize("dtype,K", [("f16", 64), ("bf16", 32), ("f32", 16)])
def test_softmax_matches_torch_sdpa(dtype, K):
    """K = L, SOFTMAX, s = 1/sqrt(K), no mask  ==  textbook scaled dot-product attention."""
    inp = gen.make_chain_inputs(21, dtype, 3, 40, 70, K, K, 1)
    A, B, D = _f64(inp)
    ours = oracle.chain(inp, "softmax", 1.0 / math.sqrt(K))
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(A), torch.from_numpy(B), torch.from_numpy(D)).numpy()
    assert np.max(np.abs(ours - ref)) < 1e-12


def test_softmax_key_padding_matches_torch_sdpa():
    inp = gen.make_chain_inputs(22, "f16", 4, 33, 90, 64, 48, 1)
    vl = np.array([90, 1, 45, 77], dtype=np.int32)
    A, B, D = _f64(inp)
    ours = oracle.chain(inp, "softmax", 0.125, valid_len=vl)
    mask = torch.arange(90)[None, None, :] < torch.from_numpy(vl)[:, None, None]
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(A), torch.from_numpy(B), torch.from_numpy(D),
        attn_mask=mask.expand(4, 33, 90), scale=0.125).numpy()
    assert np.max(np.abs(ours - ref)) < 1e-12


@pytest.mark.parametrize("M,N", [(40, 40), (33, 90), (90, 33)])
def test_causal_matches_torch_sdpa(M, N):
    """Causal mask (R18: key n visible to row m iff n <= m, top-left aligned) against
    torch SDPA's is_causal (tril(diagonal=0) of an M x N ones matrix) in fp64, square and not."""
    inp = gen.make_chain_inputs(23, "f16", 3, M, N, 64, 32, 1)
    A, B, D = _f64(inp)
    ours = oracle.chain(inp, "softmax", 0.125, causal=True)
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(A), torch.from_numpy(B), torch.from_numpy(D), is_causal=True, scale=0.125).numpy()
    assert np.max(np.abs(ours - ref)) < 1e-12


def test_causal_closed_forms_and_padding():
    """Row 0 sees key 0 only (E = D[0,:] exactly); D = ones gives E = 1; with key padding the
    limit is min(valid_len, m + 1) — a fully padded batch row stays 0; NONE ignores the flag."""
    inp = gen.make_chain_inputs(24, "bf16", 3, 50, 60, 16, 8, 1)
    E = oracle.chain(inp, "softmax", 0.5, causal=True)
    D = gen.bits_to_f64_numpy(inp.D, "bf16")
    assert np.array_equal(E[:, 0, :], D[:, 0, :])
    ones = gen.ChainInputs(inp.A, inp.B, np.full(inp.D.shape, 0x3F80, dtype=np.uint16), None, "bf16", 3, 50, 60,
                           16, 8, 1)
    assert np.max(np.abs(oracle.chain(ones, "softmax", 0.5, causal=True) - 1.0)) < 1e-12
    vl = np.array([60, 10, 0], dtype=np.int32)
    Ec = oracle.chain(inp, "softmax", 0.5, valid_len=vl, causal=True)
    A, B, _ = _f64(inp)
    for b, v in enumerate(vl):
        for m in (0, 5, 9, 10, 30, 49):
            lim = min(v, m + 1)
            if lim == 0:
                assert np.all(Ec[b, m] == 0.0)
                continue
            z = 0.5 * (A[b, m] @ B[b, :lim].T)
            p = np.exp(z - z.max())
            assert np.max(np.abs(Ec[b, m] - (p / p.sum()) @ D[b, :lim])) < 1e-12
    assert np.array_equal(oracle.chain(inp, "none", 1.0, causal=True), oracle.chain(inp, "none", 1.0))


@pytest.mark.parametrize("b_layout", [0, 1])
def test_activation_ops_through_identity_D(b_layout):
    """RELU / GELU inter-ops (R19): D = I exposes op(s·A·B) — RELU against numpy
    maximum, GELU against scipy.special.erf's definition; GELU(x) − GELU(−x) = x exactly in real
    arithmetic (checked through A → −A); GELU(0) = 0 (scale 0)."""
    from scipy.special import erf as sp_erf
    inp = gen.make_chain_inputs(35, "bf16", 2, 17, 24, 20, 24, b_layout)
    A = gen.bits_to_f64_numpy(inp.A, "bf16")
    B = gen.bits_to_f64_numpy(inp.B, "bf16")
    eye = np.broadcast_to(np.eye(24), (2, 24, 24))
    inp = _custom("bf16", A, B, eye, b_layout)
    C = A @ (B if b_layout == 0 else np.swapaxes(B, 1, 2))
    s = 0.7
    assert np.max(np.abs(oracle.chain(inp, "relu", s) - np.maximum(s * C, 0.0))) < 1e-12
    g = 0.5 * s * C * (1.0 + sp_erf(s * C / math.sqrt(2.0)))
    assert np.max(np.abs(oracle.chain(inp, "gelu", s) - g)) < 1e-12
    neg = _custom("bf16", -A, B, eye, b_layout)
    assert np.max(np.abs(oracle.chain(inp, "gelu", s) - oracle.chain(neg, "gelu", s) - s * C)) < 1e-12
    assert np.all(oracle.chain(inp, "gelu", 0.0) == 0.0)


@pytest.mark.parametrize("b_layout", [0, 1])
def test_identity_D_exposes_op(b_layout):
    """D = I (L = N)  =>  E = op(A·B): numpy matmul and scipy softmax as references."""
    inp = gen.make_chain_inputs(31, "bf16", 2, 17, 24, 20, 24, b_layout)
    eye = np.broadcast_to(np.eye(24), (2, 24, 24))
    inp = _custom("bf16", gen.bits_to_f64_numpy(inp.A, "bf16"), gen.bits_to_f64_numpy(inp.B, "bf16"),
                  eye, b_layout)
    A, B, _ = _f64(inp)
    C = A @ _bmat(inp, B)
    assert np.array_equal(oracle.chain(inp, "none"), C)
    assert np.array_equal(oracle.chain(inp, "scale", 0.25), 0.25 * C)
    sm = scipy.special.softmax(0.7 * C, axis=-1)
    assert np.max(np.abs(oracle.chain(inp, "softmax", 0.7) - sm)) < 1e-13


def test_zero_K_closed_forms():
    inp = gen.make_chain_inputs(41, "f16", 3, 5, 11, 0, 6, 1)
    assert np.array_equal(oracle.chain(inp, "none"), np.zeros((3, 5, 6)))
    assert np.array_equal(oracle.chain(inp, "scale", 2.0), np.zeros((3, 5, 6)))
    vl = np.array([11, 4, 1], dtype=np.int32)
    D = gen.bits_to_f64_numpy(inp.D, "f16")
    E = oracle.chain(inp, "softmax", 0.125, valid_len=vl)
    for b in range(3):
        ref = D[b, :vl[b]].mean(axis=0)
        assert np.max(np.abs(E[b] - ref[None, :])) < 1e-14


def test_scale_zero_is_uniform_mean():
    inp = gen.make_chain_inputs(42, "bf16", 2, 9, 19, 64, 8, 0)
    D = gen.bits_to_f64_numpy(inp.D, "bf16")
    E = oracle.chain(inp, "softmax", 0.0)
    assert np.max(np.abs(E - D.mean(axis=1)[:, None, :])) < 1e-14


def test_single_and_zero_valid_key():
    inp = gen.make_chain_inputs(43, "f16", 2, 7, 30, 64, 16, 1, sigmas=(3.0, 3.0, 1.0))
    D = gen.bits_to_f64_numpy(inp.D, "f16")
    E = oracle.chain(inp, "softmax", 0.125, valid_len=np.array([1, 0], dtype=np.int32))
    assert np.array_equal(E[0], np.broadcast_to(D[0, 0], (7, 16)))   # exactly D[0,:]
    assert np.array_equal(E[1], np.zeros((7, 16)))                    # fully masked -> 0


def test_softmax_rows_sum_to_one_and_ones_D():
    inp = gen.make_chain_inputs(44, "f16", 2, 12, 57, 64, 8, 1, sigmas=(3.0, 3.0, 1.0))
    vl = np.array([57, 20], dtype=np.int32)
    _, Cp = oracle.chain(inp, "softmax", 0.125, valid_len=vl, want_cprime=True)
    assert np.max(np.abs(Cp.sum(axis=1) - 1.0)) <= 1e-12
    assert np.all(Cp.reshape(2, 12, 57)[1, :, 20:] == 0.0)           # masked keys get 0
    ones = _custom("f16", gen.bits_to_f64_numpy(inp.A, "f16"), gen.bits_to_f64_numpy(inp.B, "f16"),
                   np.ones((2, 57, 8)), 1)
    assert np.max(np.abs(oracle.chain(ones, "softmax", 0.125, valid_len=vl) - 1.0)) <= 1e-12


def test_softmax_shift_invariance():
    """Append a K-column A[:,K]=1, B[K,:]=c: every score shifts by c*s; E is unchanged."""
    inp = gen.make_chain_inputs(45, "f32", 2, 10, 25, 16, 12, 0)
    A, B, D = _f64(inp)
    c = 3.0
    A2 = np.concatenate([A, np.ones((2, 10, 1))], axis=2)
    B2 = np.concatenate([B, np.full((2, 1, 25), c)], axis=1)
    inp2 = _custom("f32", A2, B2, D, 0)
    e1, e2 = oracle.chain(inp, "softmax", 0.25), oracle.chain(inp2, "softmax", 0.25)
    assert np.max(np.abs(e1 - e2)) < 1e-13
    # and the shift is NOT invisible to the un-normalised ops (sanity: the column is used)
    assert not np.allclose(oracle.chain(inp, "none"), oracle.chain(inp2, "none"))


def test_selected_rows_equal_full():
    inp = gen.make_chain_inputs(46, "bf16", 3, 20, 33, 48, 24, 1)
    vl = np.array([33, 10, 2], dtype=np.int32)
    full = oracle.chain(inp, "softmax", 0.2, valid_len=vl)
    rows = np.array([[0, 0], [2, 19], [1, 7], [2, 3]], dtype=np.int64)
    part = oracle.chain(inp, "softmax", 0.2, valid_len=vl, rows=rows)
    for i, (b, m) in enumerate(rows):
        assert np.array_equal(part[i], full[b, m])


def test_row_max_error_metric():
    ref = np.array([[[1.0, -2.0], [0.0, 0.0]]])
    got = np.array([[[1.0, -2.1], [0.0, 0.5]]])
    # row 0: 0.1/2 = 0.05; row 1: all-zero reference -> absolute 0.5
    assert oracle.row_max_error(got, ref) == pytest.approx(0.5)
    assert oracle.row_max_error(got[:, :1], ref[:, :1]) == pytest.approx(0.05)
    assert math.isnan(oracle.row_max_error(np.full_like(ref, np.nan), ref))


# ---------------------------------------------------------------- paper numbers
def _read_golden(name):
    rows = []
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#", 1)[0].strip()
        if line:
            rows.append(line)
    return rows


def test_phi_goldens():
    for line in _read_golden("phi.txt"):
        f, TM, TN, K, exp, tol = line.split()
        got = getattr(model, f)(float(TM), float(TN), float(K))
        assert abs(got - float(exp)) <= float(tol), line
    # the two readings round to the paper's "227 to 2" only for phi_text
    assert round(model.phi_text(256, 256, 1024)) == 228 and int(model.phi_text(256, 256, 1024)) == 227
    assert round(model.phi_text(256, 256, 1)) == 2
    assert round(model.phi_printed(256, 256, 1)) == 1


def test_is_memory_bound_examples():
    """PAPER.md:119 (§II-A): MBCI iff φ < P/W (strict).  SPEC.md:76-79 examples: threshold 100
    flops per element, φ = 204.8 → compute-bound, φ = 0.996 → memory-bound, φ == P/W →
    compute-bound."""
    W = 1.0e12
    P = 100.0 * W   # P / W = 100
    assert not model.is_memory_bound(model.phi_printed(256, 256, 1024), P, W)
    assert model.is_memory_bound(model.phi_printed(256, 256, 1), P, W)
    assert not model.is_memory_bound(100.0, P, W)
    assert model.is_memory_bound(math.nextafter(100.0, 0.0), P, W)
    # §I's narrative: K 1024 → 1 moves a 256-tile MatMul across any threshold
    # between the two ratios, e.g. A100's FP16 ridge 312e12 / 1.555e12 ≈ 200.6 flops per byte
    ridge = 312e12 / 1.555e12
    assert not model.is_memory_bound(model.phi_text(256, 256, 1024), ridge, 1.0)
    assert model.is_memory_bound(model.phi_text(256, 256, 1), ridge, 1.0)


def test_fused_intensity_independent_of_K_L():
    for K, L in ((16, 16), (64, 64), (128, 32)):
        assert model.fused_intensity(512, 512, K, L, 2) == pytest.approx(256.0)
    assert model.fused_intensity(256, 256, 64, 64, 2) == pytest.approx(128.0)
    assert model.fused_intensity(1024, 256, 64, 80, 2) == pytest.approx(2 * 1024 * 256 / (1280 * 2))


def test_model_goldens():
    g = {}
    for line in _read_golden("model.txt"):
        lhs, rhs = line.split("=")
        g[lhs.strip()] = float(rhs)
    assert len(model.deep_expressions()) == g["deep_count"]
    assert len(set(model.deep_expressions())) == 24
    assert len(model.flat_expressions()) == g["flat_count"]
    assert model.space_size(1024, 1024, 512, 512) == g["space_size 1024 1024 512 512"]
    assert model.space_size(64, 64, 32, 32) == g["space_size 64 64 32 32"]
    assert model.alpha(108, 108) == g["alpha 108 108"]
    assert model.alpha(1, 108) == g["alpha 1 108"]
    assert model.alpha(10**6, 108) == pytest.approx(g["alpha 1000000 108"], abs=1e-12)
    assert model.t_mem([(64 * 64 * 2, [4, 2])], 1e9) == pytest.approx(g["t_mem_single_load"], rel=1e-12)
    assert model.t_comp([(2 * 64**3, [4, 4, 2])], 1e12) == pytest.approx(g["t_comp_single_compute"], rel=1e-12)
    assert model.shm_estm([(64, 64)] * 5) * 2 == g["shm_estm_five_64x64_fp16"]
    assert not model.rule4_reject(40960, 48 * 1024)
    assert model.rule4_reject(100000, 65536)
    assert model.t_estm(6.5536e-5, 1.6777216e-5, 2.0) == pytest.approx(2 * (6.5536e-5 + 1.6777216e-5))


def test_rule3_and_tile_options():
    assert model.rule3_reject(1024, 48)          # power of 2, padded
    assert not model.rule3_reject(1000, 48)      # 8/1000 < 0.05
    assert not model.rule3_reject(1024, 64)
    assert model.rule3_reject(100, 48)           # 44/100 >= 0.05
    assert model.tile_options(40) == [16, 32, 48]
    assert model.tile_options(16) == [16]


def test_chain_schedule_dead_loop_and_hoist():
    """with k dead, L_A executes l_m times instead of l_m*l_h*l_n*l_k;
    PAPER.md:232: S_E is hoisted out of n (trip l_m*l_h)."""
    mem, comp, nb = model.chain_schedule(1, 512, 512, 64, 64, 128, 128, 64, 64, 2)
    la, lb, ld, se = mem
    assert math.prod(la[1]) == 4            # l_m, dead k
    assert math.prod(lb[1]) == 4 * 1 * 4 * 1
    assert math.prod(se[1]) == 4            # not multiplied by l_n = 4
    mem2, _, _ = model.chain_schedule(1, 512, 512, 128, 64, 128, 128, 64, 64, 2)
    assert math.prod(mem2[0][1]) == 4 * 1 * 4 * 2   # live k: L_A under m,h,n,k
    # total FLOPs do not depend on TM/TN: 2MN(K+L) per batch when h is dead ...
    for TN in (64, 128, 256):
        _, comp, _ = model.chain_schedule(2, 512, 512, 64, 64, 128, TN, 64, 64, 2)
        assert sum(fp * math.prod(lp) for fp, lp in comp) == 2 * 2 * 512 * 512 * 128
    # ... while chunking L onto the grid (l_h = 2) recomputes C_C l_h times
    _, comp, _ = model.chain_schedule(2, 512, 512, 64, 64, 128, 128, 64, 32, 2)
    assert sum(fp * math.prod(lp) for fp, lp in comp) == 2 * 2 * 512 * 512 * (2 * 64 + 64)
    # hoisted bytes equal the algorithmic (M+N)(K+L)s per batch when every tile covers its dim
    mem, _, _ = model.chain_schedule(1, 256, 256, 64, 64, 256, 256, 64, 64, 2)
    assert sum(ts * math.prod(lp) for ts, lp in mem) == (256 + 256) * (64 + 64) * 2


# ---------------------------------------------------------------- three contractions (R20)
def test_chain3_identity_F_and_reassociation():
    """oracle.chain3: F = I (H = L) gives op2 of the two-contraction chain exactly; NONE / NONE on
    integer inputs equals the two-contraction chain with D·F (exact integer arithmetic)."""
    inp = gen.make_chain_inputs(51, "bf16", 2, 9, 13, 7, 6, 1)
    eye = np.broadcast_to(np.eye(6), (2, 6, 6))
    Fi = (np.asarray(eye, np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    E2 = oracle.chain(inp, "softmax", 0.4)
    assert np.array_equal(oracle.chain3(inp, Fi, 6, "softmax", 0.4, "none"), E2)
    assert np.array_equal(oracle.chain3(inp, Fi, 6, "softmax", 0.4, "relu", 1.0), np.maximum(E2, 0.0))
    assert np.array_equal(oracle.chain3(inp, Fi, 6, "softmax", 0.4, "scale", -2.0), -2.0 * E2)
    ii = gen.make_chain_inputs(52, "f16", 2, 5, 7, 4, 3, 0, kind="int")
    F = gen.make_chain_inputs(53, "f16", 2, 3, 1, 5, 1, 0, kind="int").A   # [2, L=3, H=5] (A's [b, M, K] shape)
    D = gen.bits_to_f64_numpy(ii.D, "f16")
    DF = D @ gen.bits_to_f64_numpy(F, "f16")                          # |DF| <= 12: exact in fp16
    ii2 = gen.ChainInputs(ii.A, ii.B, gen._f64_to_storage(DF.ravel(), "f16").reshape(2, 7, 5), None, "f16", 2, 5,
                          7, 4, 5, 0)
    assert np.array_equal(oracle.chain3(ii, F, 5, "none", 1.0, "none"), oracle.chain(ii2, "none", 1.0))


def test_chain3_brute_force_numpy():
    inp = gen.make_chain_inputs(54, "f16", 3, 6, 10, 5, 4, 1, valid_len_range=(1, 10))
    F = gen.make_chain_inputs(55, "f16", 3, 4, 1, 7, 1, 1).A   # [3, L=4, H=7]
    A = gen.bits_to_f64_numpy(inp.A, "f16")
    B = gen.bits_to_f64_numpy(inp.B, "f16")
    D = gen.bits_to_f64_numpy(inp.D, "f16")
    Ff = gen.bits_to_f64_numpy(F, "f16")
    from scipy.special import erf as sp_erf
    for causal in (False, True):
        got = oracle.chain3(inp, F, 7, "softmax", 0.3, "gelu", 1.7, valid_len=inp.valid_len, causal=causal)
        for b in range(3):
            for m in range(6):
                lim = min(int(inp.valid_len[b]), m + 1) if causal else int(inp.valid_len[b])
                z = 0.3 * (A[b, m] @ B[b, :lim].T)
                p = np.exp(z - z.max())
                e = (p / p.sum()) @ D[b, :lim]
                g = 0.5 * 1.7 * e * (1.0 + sp_erf(1.7 * e / math.sqrt(2.0)))
                assert np.max(np.abs(got[b, m] - g @ Ff[b])) < 1e-12


# ---- Fig. 7 pruning funnel (§III-C) -------------------------------------------------
def _funnel_golden():
    g = {}
    for line in _read_golden("funnel.txt"):
        lhs, rhs = line.split("=")
        g[lhs.strip()] = rhs.strip()
    return g


def test_funnel_rule1_rule2_against_paper_examples():
    g = _funnel_golden()
    a, b, key = g["rule1_same_class"].split()
    assert model.sub_tiling_expression(a) == key == model.sub_tiling_expression(b)
    assert model.sub_tiling_expression("mhkn") == g["rule2_rejected_class"]   # Fig. 6 caption: "kn"
    assert model.rule2_reject(g["rule2_rejected_class"])
    assert not model.rule2_reject(key)
    # every deep permutation keeps n and k in its own order; both flat ones keep n outside k
    for e in model.deep_expressions():
        k = model.sub_tiling_expression(e)
        assert k == ("nk" if e.index("n") < e.index("k") else "kn")
    assert {model.sub_tiling_expression(e) for e in model.flat_expressions()} == {"n(k)"}


def test_funnel_counts_against_paper():
    g = _funnel_golden()
    f = model.prune_funnel(1024, 1024, 512, 512, 2, 166912)   # A100 (the paper's platform): 163 KB
    assert f["raw"] == int(g["raw_candidates"])
    assert f["expr_raw"] == int(g["expressions"])
    assert f["expr_rule1"] == 3 and f["expr_rule2"] == 2 and f["keys"] == ["nk", "kn", "n(k)"]
    # Rule 3 on power-of-2 dims keeps exactly the power-of-2 tiles 16 .. dim (closed form)
    closed = 1
    for d in (1024, 1024, 512, 512):
        closed *= int(math.log2(d // 16)) + 1
    assert f["tile_vectors_rule3"] == closed == 7 * 7 * 6 * 6
    assert 1 - f["tile_vectors_rule3"] / f["tile_vectors"] >= float(g["rule3_min_discard"])
    assert int(g["final_order_low"]) <= f["after_rule4"] <= int(g["final_order_high"])
    # Rule 4 brute force: Eq. (1) over the 1764 survivors by plain loops
    surv = [[t for t in model.tile_options(d) if not model.rule3_reject(d, t)] for d in (1024, 1024, 512, 512)]
    kept = sum(1 for tm in surv[0] for tn in surv[1] for tk in surv[2] for th in surv[3]
               if not model.rule4_reject(model.shm_estm([(tm, tk), (tk, tn), (tm, tn), (tn, th), (tm, th)]) * 2, 166912))
    assert f["tile_vectors_rule4"] == kept


def test_funnel_limits_and_ragged_dims():
    # Rule 4 with an unbounded budget rejects nothing, with a 1-byte budget everything
    f = model.prune_funnel(256, 256, 64, 64, 2, 10**12)
    assert f["tile_vectors_rule4"] == f["tile_vectors_rule3"]
    assert model.prune_funnel(256, 256, 64, 64, 2, 1)["tile_vectors_rule4"] == 0
    # SPEC.md:158 tiny space: 26 x 4*4*2*2
    assert model.prune_funnel(64, 64, 32, 32, 2, 232448)["raw"] == 1664
    # ragged dim 1000 (not a power of 2): a tile survives iff its padding is < 50 elements
    keep = [t for t in model.tile_options(1000) if not model.rule3_reject(1000, t)]
    assert keep == [t for t in range(16, 1009, 16) if math.ceil(1000 / t) * t - 1000 < 50]
    assert 1008 in model.tile_options(1000) and 1008 in keep   # 8 / 1000 padding


# ---- split-N statistic: the row log-sum-exp -----------------------------------
def test_row_lse_against_scipy_logsumexp():
    from split_util import slice_keys  # noqa: F401
    inp = gen.make_chain_inputs(11, "bf16", 3, 9, 21, 16, 8, 1, valid_len_range=(0, 21))
    A, B, _ = _f64(inp)
    s = 0.37
    z = s * np.einsum("bmk,bkn->bmn", A, _bmat(inp, B))
    for vl in (None, inp.valid_len):
        got = oracle.row_lse(inp, s, vl)
        for b in range(inp.batch):
            v = inp.N if vl is None else int(vl[b])
            ref = scipy.special.logsumexp(z[b, :, :v], axis=1) if v > 0 else np.full(inp.M, -np.inf)
            assert np.allclose(got[b], ref, rtol=0, atol=1e-12) or (v == 0 and np.all(got[b] == -np.inf))
    # one valid key: lse = s * C[m, 0] exactly; no valid key: -inf
    got = oracle.row_lse(inp, s, np.array([1, 0, 21], dtype=np.int32))
    assert np.allclose(got[0], z[0, :, 0], rtol=0, atol=1e-12)
    assert np.all(got[1] == -np.inf)


@pytest.mark.parametrize("cuts", [(0, 7, 21), (0, 1, 2, 21), (0, 20, 21), (0, 8, 16, 21)])
@pytest.mark.parametrize("masked", [False, True])
def test_split_n_combination_reproduces_full_chain(cuts, masked):
    """Partial chains over key ranges, combined by log-sum-exp weights, equal the full chain: the
    identity the GPU merge (mbci_merge_partials) implements, checked on the oracle alone."""
    from split_util import local_valid, lse_combine, slice_keys
    inp = gen.make_chain_inputs(12, "f16", 4, 10, 21, 16, 12, 1, valid_len_range=(0, 21) if masked else None)
    vl = inp.valid_len if masked else None
    s = 0.25
    full = oracle.chain(inp, "softmax", s, vl)
    parts, lses = [], []
    for n0, n1 in zip(cuts, cuts[1:]):
        sub = slice_keys(inp, n0, n1)
        v = local_valid(vl, n0, n1)
        parts.append(oracle.chain(sub, "softmax", s, v))
        lses.append(oracle.row_lse(sub, s, v))
    assert np.allclose(lse_combine(parts, lses), full, rtol=0, atol=1e-12)
    # linear ops: the partial products simply add up
    full_none = oracle.chain(inp, "none", 1.0)
    parts = [oracle.chain(slice_keys(inp, a, b), "none", 1.0) for a, b in zip(cuts, cuts[1:])]
    assert np.allclose(np.sum(parts, axis=0), full_none, rtol=0, atol=1e-10)
