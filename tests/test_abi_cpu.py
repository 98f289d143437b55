"""C-ABI contract checks that need no GPU: the library loads, exports every symbol the
header declares, validates descriptors, and its host-only tile selector reproduces the
paper's model (oracle/model.py) and respects the B200 budgets."""
import ctypes
import math
import os
import re
import subprocess

import pytest

from oracle import model

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mbci.h")


@pytest.fixture(scope="module")
def m():
    from paper_2506_22169_b200 import _build
    _build.build()
    from paper_2506_22169_b200 import mbci
    return mbci


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mbci_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_header_symbol(m):
    names = header_functions()
    assert len(names) >= 14
    out = subprocess.run(["nm", "-D", "--defined-only", m.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b[TW] (mbci_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert hasattr(m._lib, n)
    assert sorted(m.EXPORTED) == names


def test_version_and_status_strings(m):
    assert m.mbci_abi_version() == 1
    assert m.mbci_status_string(0) == b"MBCI_OK"
    assert m.mbci_status_string(2) == b"MBCI_ERR_UNSUPPORTED"


def _create(m, d):
    h = ctypes.c_void_p()
    return m.mbci_chain_create(ctypes.byref(d) if d is not None else None, 0, ctypes.byref(h)), h


def test_validation_errors(m):
    assert _create(m, None)[0] == m.MBCI_ERR_INVALID
    assert _create(m, m.make_desc(-1, 8, 8, 8, 8))[0] == m.MBCI_ERR_INVALID
    d = m.make_desc(1, 8, 8, 8, 8)
    d.dtype = 7
    assert _create(m, d)[0] == m.MBCI_ERR_INVALID
    d = m.make_desc(1, 8, 8, 8, 8, op="none", mask=True)
    assert _create(m, d)[0] == m.MBCI_ERR_INVALID
    assert _create(m, m.make_desc(1, 8, 8, 65537, 8))[0] == m.MBCI_ERR_UNSUPPORTED    # K, L <= 65536
    assert _create(m, m.make_desc(1, 8, 8, 64, 65537))[0] == m.MBCI_ERR_UNSUPPORTED
    d = m.make_desc(1, 8, 8, 16, 8, strides={"ld_a": 8})   # row stride shorter than the row
    assert _create(m, d)[0] == m.MBCI_ERR_INVALID
    assert b"stride" in m.mbci_last_error()
    assert m.mbci_chain_run(None, None, None, None, None, None, None) == m.MBCI_ERR_INVALID
    assert m.mbci_chain_destroy(None) == m.MBCI_OK


def test_no_gpu_reports_cuda_error(m):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st, h = _create(m, m.make_desc(2, 128, 128, 64, 64, "f16"))
    assert st in (m.MBCI_ERR_CUDA, m.MBCI_ERR_INVALID)
    assert not h.value


# ---------------------------------------------------------------- selector vs paper model
SHAPES = [(96, 512, 512, 64, 64), (128, 1024, 1024, 64, 64), (64, 2048, 2048, 16, 16),
          (64, 2048, 2048, 128, 128), (1, 128, 128, 16, 16), (3, 1000, 777, 80, 80),
          (8, 1024, 1024, 128, 128), (1, 512, 256, 64, 128)]


@pytest.mark.parametrize("shape", SHAPES)
def test_model_terms_match_oracle(m, shape):
    b, M, N, K, L = shape
    hw = m.hw_default()
    for TM, TN, TK, TH in [(128, 128, 64, 64), (128, 64, 16, 32), (64, 256, 128, 16), (16, 16, 16, 16),
                           (256, 128, 32, 128)]:
        got = m.model_terms(b, M, N, K, L, TM, TN, TK, TH, 2, hw)
        ref = model.chain_estimate(b, M, N, K, L, TM, TN, TK, TH, 2, hw.W, hw.P, hw.n_sm)
        for k in ("t_mem", "t_comp", "alpha", "t_estm", "n_block"):
            assert got[k] == pytest.approx(ref[k], rel=1e-12), (k, TM, TN, TK, TH)


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("b_layout", [0, 1])
def test_enumerated_plans_are_legal_and_scored(m, shape, b_layout):
    b, M, N, K, L = shape
    hw = m.hw_default()
    d = m.make_desc(b, M, N, K, L, "bf16", "softmax", b_layout=b_layout)
    st, plans = m.plan_enumerate(d, hw)
    assert st == m.MBCI_OK and plans
    lpad = max(16, math.ceil(L / 16) * 16)
    rule3_ok = any(not model.rule3_reject(N, bn) for bn in (64, 128))
    scores = [p.t_b200 for p in plans]
    assert scores == sorted(scores)
    b_inner = N if b_layout == 0 else K
    if any(x % 8 for x in (K, b_inner, L)):        # TMA needs 16-byte row strides
        assert [p.kernel for p in plans] == [1]
        return
    assert {p.kernel for p in plans} <= {0, 4, 5, 6}
    for p in plans:
        assert p.kernel in (0, 4, 5, 6) and p.BN in (64, 128)
        assert p.BM == (256 if p.kernel >= 4 else 128)   # kernels 4-6: two 128-row Q tiles per CTA
        if p.kernel >= 4:    # whole L in the CTA, 128-key tiles
            assert p.TL == lpad and p.BN == 128
        if p.kernel >= 5:         # S_0, S_1 + P_0, P_1 + O_0, O_1 in 512 TMEM columns
            assert p.TL <= 64
        assert p.TL % 16 == 0 and 16 <= p.TL <= lpad
        assert p.TK == max(16, math.ceil(K / 16) * 16)
        assert p.smem_bytes <= hw.smem_max
        if p.kernel == 0:    # one CTA pipeline: S double-buffered + O
            assert 2 * p.BN + p.TL <= p.tmem_cols <= 512 and p.tmem_cols & (p.tmem_cols - 1) == 0
        else:
            assert p.tmem_cols == 512 and p.smem_bytes + 5120 <= hw.smem_max
        assert 2 <= p.stages <= (4 if p.kernel == 0 else 8)
        if rule3_ok and p.kernel == 0:   # kernels 4 / 5 mask ragged key tiles: exempt from Rule 3
            assert not model.rule3_reject(N, p.BN)
        ref = model.chain_estimate(b, M, N, K, L, p.BM, p.BN, p.TK, p.TL, 2, hw.W, hw.P, hw.n_sm)
        assert p.t_estm == pytest.approx(ref["t_estm"], rel=1e-12)
        assert p.alpha == pytest.approx(ref["alpha"], rel=1e-12)
        assert p.n_block == b * math.ceil(M / p.BM) * math.ceil(L / p.TL)
    best = m.mbci_plan_t()
    assert m.mbci_plan_select(ctypes.byref(d), ctypes.byref(hw), ctypes.byref(best)) == m.MBCI_OK
    assert best.t_b200 == plans[0].t_b200


def test_bert_base_prefers_full_L_tile(m):
    """Chunking L onto the grid recomputes C; with 384 CTAs already
    filling the GPU the selector keeps T_H = L."""
    d = m.make_desc(96, 512, 512, 64, 64, "f16", "softmax")
    p = m.mbci_plan_t()
    assert m.mbci_plan_select(ctypes.byref(d), None, ctypes.byref(p)) == m.MBCI_OK
    assert p.TL == 64 and p.kernel in (0, 4, 5, 6)


def test_fp32_goes_to_tf32x3_tensor_cores_and_misaligned_to_cuda_cores(m):
    """fp32 (north_star (3)): kernel 7 (tcgen05 kind::tf32, 3xTF32) first whenever 1 <= K, L <= 128,
    the CUDA-core kernel 1 behind it as the fallback; 16-bit rows that break TMA's 16-B rule and fp32
    shapes outside kernel 7 go to kernel 1 only."""
    st, plans = m.plan_enumerate(m.make_desc(1, 128, 128, 16, 16, "f32", "none"))
    assert st == m.MBCI_OK and [p.kernel for p in plans] == [7, 1]
    assert plans[0].BM == 128 and plans[0].BN == 64 and plans[0].TK == 16 and plans[0].TL == 16
    st, plans = m.plan_enumerate(m.make_desc(3, 300, 200, 20, 40, "f32", "softmax", 0.2))
    assert st == m.MBCI_OK and [p.kernel for p in plans] == [7, 1] and plans[0].TK == 24 and plans[0].TL == 48
    for K, L in ((80, 16), (16, 80), (128, 128)):   # the wide variant: 32-key tiles, 128 O columns
        st, plans = m.plan_enumerate(m.make_desc(1, 128, 128, K, L, "f32", "none"))
        assert st == m.MBCI_OK and [p.kernel for p in plans] == [7, 1] and plans[0].BN == 32
    for K, L in ((136, 16), (16, 136), (0, 16)):
        st, plans = m.plan_enumerate(m.make_desc(1, 128, 128, K, L, "f32", "none"))
        assert st == m.MBCI_OK and [p.kernel for p in plans] == [1]
    st, plans = m.plan_enumerate(m.make_desc(2, 3, 5, 3, 3, "f16", "none"))   # K=3: 6-byte rows
    assert st == m.MBCI_OK and plans[0].kernel == 1
    st, plans = m.plan_enumerate(m.make_desc(1, 16, 10**6, 16, 16, "f32", "none"))  # C row > SMEM: kernel 7 only
    assert st == m.MBCI_OK and [p.kernel for p in plans] == [7]
    st, plans = m.plan_enumerate(m.make_desc(1, 16, 10**6, 16, 136, "f32", "none"))
    assert st == m.MBCI_ERR_UNSUPPORTED and plans == []


def test_rule3_fallback_keeps_a_plan_on_ragged_N(m):
    """N = 300: every BN pads >= 5 % (Rule 3 rejects all); the selector then skips the rule."""
    st, plans = m.plan_enumerate(m.make_desc(2, 200, 300, 64, 64, "bf16"))
    assert st == m.MBCI_OK and plans
    assert all(model.rule3_reject(300, p.BN) for p in plans)


def test_persistent_plans_for_attention_shapes(m):
    """Kernel 5 (separate P) is the default for 16-bit chains with L <= 64 and kernel 4 for
    64 < L <= 128, for every op; their plans use the whole L per CTA, 128-key tiles, fit SMEM
    with room for the static (l, m) arrays, and the 4-stage plan (which enables half items for
    the last partial round) ranks first on C2."""
    hw = m.hw_default()
    for op in ("softmax", "scale", "none"):
        d = m.make_desc(96, 512, 512, 64, 64, "f16", op, 0.125)
        st, plans = m.plan_enumerate(d, hw)
        assert st == m.MBCI_OK and plans[0].kernel == 5
    d = m.make_desc(96, 512, 512, 64, 64, "f16", "softmax", 0.125)
    st, plans = m.plan_enumerate(d, hw)
    for kern in (4, 5):
        kp = [p for p in plans if p.kernel == kern]
        assert kp[0].stages == 4
        assert all(p.stages >= (3 if kern == 4 else 2) for p in kp)
        by_stages = {p.stages: p.t_b200 for p in kp}
        assert by_stages[4] < by_stages[3]          # half items (stages >= 4) halve the tail round
        for p in kp:
            assert p.BN == 128 and p.TL == 64 and p.BM == 256 and p.tmem_cols == 512
            assert p.smem_bytes + 5120 <= hw.smem_max
    # key padding disables half items: the 3- and 4-stage plans then score alike
    d = m.make_desc(96, 512, 512, 64, 64, "f16", "softmax", 0.125, mask=True)
    st, plans = m.plan_enumerate(d, hw)
    k5 = {p.stages: p.t_b200 for p in plans if p.kernel == 5}
    assert abs(k5[4] - k5[3]) < 1e-9
    # d = 128 (C5 shape): kernel 4 with two S buffers; a 2-deep ring is the only fit with the Q pair
    d = m.make_desc(512, 4096, 4096, 128, 128, "bf16", "softmax", 0.125)
    st, plans = m.plan_enumerate(d, hw)
    assert plans[0].kernel == 4 and plans[0].stages == 2 and plans[0].TL == 128
    assert not any(p.kernel in (5, 6) for p in plans)


@pytest.mark.parametrize("N", [192, 320, 448, 576, 960, 1000, 512])
def test_persistent_kernel_default_on_any_N(m, N):
    """Rule 3 prunes kernel 0's BN only: the persistent kernels mask the ragged
    last 128-key tile, so an odd multiple of 64 (or any N) keeps them as the default."""
    st, plans = m.plan_enumerate(m.make_desc(96, 512, N, 64, 64, "f16", "softmax", 0.125))
    assert st == m.MBCI_OK and plans[0].kernel == 5
    st, plans = m.plan_enumerate(m.make_desc(512, 512, N, 128, 128, "bf16", "softmax", 0.125))
    assert st == m.MBCI_OK and plans[0].kernel == 4
    st, plans = m.plan_enumerate(m.make_desc(4, 256, N, 128, 128, "bf16", "softmax", 0.125))
    assert {4, 0} <= {p.kernel for p in plans}     # a candidate even where kernel 0 ranks first


@pytest.mark.parametrize("K,L", [(256, 256), (512, 256), (1024, 256), (64, 256), (136, 64), (4096, 136)])
def test_large_K_L_plans_are_kernel0_with_live_k_loop_or_h_chunks(m, K, L):
    """SURVEY §8(f) f3 (Table II G3-G6): K > 128 streams A and B in 64-column chunks
    (ring entry = 16 KB A chunk + BN x 128 B B chunk, no resident A), L > 128 is cut into h chunks
    of TL <= 128 columns; only kernel 0 takes these shapes, and every plan fits SMEM and TMEM."""
    hw = m.mbci_hw_t()
    m.mbci_hw_default(ctypes.byref(hw))
    st, plans = m.plan_enumerate(m.make_desc(1, 512, 512, K, L, "f16", "none", 1.0, b_layout=0), hw)
    assert st == m.MBCI_OK and plans and all(p.kernel == 0 for p in plans)
    for p in plans:
        assert p.TL <= 128 and p.TL % 16 == 0 and p.smem_bytes <= hw.smem_max
        assert 2 * p.BN + p.TL <= 512
        if K > 128:   # no resident A: stages x (A chunk + B chunk) + stages x D stage + barriers
            dch = (p.TL + 63) // 64
            assert p.smem_bytes >= p.stages * (16384 + p.BN * 128 + dch * p.BN * 128)
    fp32 = m.plan_enumerate(m.make_desc(1, 512, 512, K, L, "f32", "none", 1.0))[1]
    assert [p.kernel for p in fp32] == ([7, 1] if K <= 128 and L <= 128 else [1])


@pytest.mark.parametrize("shape", [(1024, 1024, 512, 512), (64, 64, 32, 32), (1000, 1000, 500, 500),
                                   (512, 512, 64, 64), (4096, 4096, 128, 128), (197, 197, 64, 64)])
@pytest.mark.parametrize("shm", [101376, 166912, 232448])
def test_prune_funnel_matches_oracle(m, shape, shm):
    """mbci_prune_funnel (csrc/prune.cpp) against oracle.model.prune_funnel (Fig. 7)."""
    from oracle import model
    got = m.prune_funnel(*shape, 2, shm)
    ref = model.prune_funnel(*shape, 2, shm)
    for k, v in got.items():
        assert v == ref[k], (k, v, ref[k])


def test_prune_funnel_errors(m):
    f = m.mbci_funnel_t()
    assert m.mbci_prune_funnel(0, 1, 1, 1, 2, 1000, ctypes.byref(f)) == 1
    assert m.mbci_prune_funnel(16, 16, 16, 16, 2, 1000, None) == 1


def test_linear_ops_prefer_deepest_ring_with_two_q_buffers(m):
    """Kernel 5 on plain chains: the deepest K/V ring that keeps both Q buffers (C4 K = L = 16: 7
    stages, measured 44.8 -> 43.0 us vs 4); softmax keeps 4 stages (short items need two Q buffers)."""
    for (K, L, op, st) in [(16, 16, "none", 7), (32, 32, "none", 5), (64, 64, "none", 4), (64, 64, "softmax", 4)]:
        d = m.make_desc(64, 2048, 2048, K, L, "bf16", op, 0.125, b_layout=0 if op == "none" else 1)
        p = m.mbci_plan_t()
        m.check(m.mbci_plan_select(d, None, p))
        assert p.kernel == 5 and p.stages == st, (K, L, op, p.kernel, p.stages)
