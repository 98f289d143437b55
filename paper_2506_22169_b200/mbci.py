"""ctypes binding of include/mbci.h — argument marshalling only.

Every step of the chain runs in libmbci.so's CUDA kernels; this module never computes
any part of it.  If the library is missing, importing this module raises (there is no
CPU fallback).  The same names as the C ABI are exported, plus a small ``Chain``
wrapper that takes torch tensors (torch is used for device memory and streams only).
"""
from __future__ import annotations

import ctypes
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MBCI_LIB: unset -> libmbci.so; "trace" -> libmbci_trace.so (diagnostics build); "ab:<name>" -> an
# A/B copy <name> next to libmbci.so (tools only; bench.py echoes MBCI_* in its JSON line)
_lib_sel = os.environ.get("MBCI_LIB", "")
LIB_PATH = os.path.join(HERE, "libmbci_trace.so" if _lib_sel == "trace"
                        else (_lib_sel[3:] if _lib_sel.startswith("ab:") else "libmbci.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the chain has no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

MBCI_F32, MBCI_F16, MBCI_BF16 = 0, 1, 2
MBCI_OP_NONE, MBCI_OP_SCALE, MBCI_OP_SOFTMAX = 0, 1, 2
MBCI_MASK_NONE, MBCI_MASK_KEY_PADDING, MBCI_MASK_CAUSAL, MBCI_MASK_CAUSAL_KEY_PADDING = 0, 1, 2, 3
MBCI_OK, MBCI_ERR_INVALID, MBCI_ERR_UNSUPPORTED, MBCI_ERR_CUDA, MBCI_ERR_NOMEM = 0, 1, 2, 3, 4

DTYPES = {"f32": MBCI_F32, "f16": MBCI_F16, "bf16": MBCI_BF16}
MBCI_OP_RELU, MBCI_OP_GELU = 3, 4
OPS = {"none": MBCI_OP_NONE, "scale": MBCI_OP_SCALE, "softmax": MBCI_OP_SOFTMAX, "relu": MBCI_OP_RELU,
       "gelu": MBCI_OP_GELU}


class mbci_chain_desc_t(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("M", ctypes.c_int64), ("N", ctypes.c_int64),
                ("K", ctypes.c_int64), ("L", ctypes.c_int64), ("dtype", ctypes.c_int32),
                ("op", ctypes.c_int32), ("scale", ctypes.c_float), ("mask", ctypes.c_int32),
                ("b_layout", ctypes.c_int32), ("ld_a", ctypes.c_int64), ("ld_b", ctypes.c_int64),
                ("ld_d", ctypes.c_int64), ("ld_e", ctypes.c_int64), ("bs_a", ctypes.c_int64),
                ("bs_b", ctypes.c_int64), ("bs_d", ctypes.c_int64), ("bs_e", ctypes.c_int64),
                ("tune", ctypes.c_int32)]


class mbci_hw_t(ctypes.Structure):
    _fields_ = [("W", ctypes.c_double), ("P", ctypes.c_double), ("n_sm", ctypes.c_int32),
                ("smem_max", ctypes.c_int32), ("tmem_cols", ctypes.c_int32),
                ("sfu_per_clk_sm", ctypes.c_double), ("clock_hz", ctypes.c_double)]


class mbci_plan_t(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("BM", ctypes.c_int32), ("BN", ctypes.c_int32),
                ("TK", ctypes.c_int32), ("TL", ctypes.c_int32), ("stages", ctypes.c_int32),
                ("smem_bytes", ctypes.c_int32), ("tmem_cols", ctypes.c_int32),
                ("n_block", ctypes.c_int64), ("t_mem", ctypes.c_double), ("t_comp", ctypes.c_double),
                ("alpha", ctypes.c_double), ("t_estm", ctypes.c_double), ("t_b200", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_P = ctypes.POINTER
_vp = ctypes.c_void_p
_st = ctypes.c_int

_lib.mbci_chain_create.argtypes = [_P(mbci_chain_desc_t), ctypes.c_int, _P(_vp)]
_lib.mbci_chain_create_with_plan.argtypes = [_P(mbci_chain_desc_t), ctypes.c_int, _P(mbci_plan_t), _P(_vp)]
_lib.mbci_chain_run.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.mbci_chain_run_host.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.mbci_chain_destroy.argtypes = [_vp]
_lib.mbci_chain_plan.argtypes = [_vp, _P(mbci_plan_t)]
_lib.mbci_chain_describe.argtypes = [_vp, ctypes.c_char_p, ctypes.c_size_t]
_lib.mbci_chain_set_trace.argtypes = [_vp, _vp, ctypes.c_int64]
_lib.mbci_chain_launches_per_run.argtypes = [_vp]
_lib.mbci_chain_launches_per_run.restype = ctypes.c_int32
_lib.mbci_status_string.argtypes = [ctypes.c_int]
_lib.mbci_status_string.restype = ctypes.c_char_p
_lib.mbci_last_error.restype = ctypes.c_char_p
_lib.mbci_abi_version.restype = ctypes.c_int32
_lib.mbci_hw_default.argtypes = [_P(mbci_hw_t)]
_lib.mbci_hw_default.restype = None
_lib.mbci_plan_enumerate.argtypes = [_P(mbci_chain_desc_t), _P(mbci_hw_t), _P(mbci_plan_t), ctypes.c_int32,
                                     _P(ctypes.c_int32)]
_lib.mbci_plan_select.argtypes = [_P(mbci_chain_desc_t), _P(mbci_hw_t), _P(mbci_plan_t)]
_lib.mbci_model_terms.argtypes = [ctypes.c_int64] * 9 + [ctypes.c_int32, _P(mbci_hw_t), _P(ctypes.c_double)]


class mbci_search_params_t(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("n", ctypes.c_int32), ("eps", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("max_rounds", ctypes.c_int32), ("model", ctypes.c_int32)]


class mbci_search_result_t(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int32), ("measurements", ctypes.c_int32), ("space_size", ctypes.c_int32),
                ("best_measured", ctypes.c_double), ("history_min", ctypes.c_double)]


class mbci_chain3_desc_t(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("M", ctypes.c_int64), ("N", ctypes.c_int64), ("K", ctypes.c_int64),
                ("L", ctypes.c_int64), ("H", ctypes.c_int64), ("dtype", ctypes.c_int32), ("op", ctypes.c_int32),
                ("scale", ctypes.c_float), ("mask", ctypes.c_int32), ("b_layout", ctypes.c_int32),
                ("op2", ctypes.c_int32), ("scale2", ctypes.c_float)]


_lib.mbci_chain_run_partial.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp]
_lib.mbci_merge_partials.argtypes = [ctypes.c_int32, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int32, ctypes.c_int32, _vp]
_lib.mbci_chain3_create.argtypes = [_P(mbci_chain3_desc_t), ctypes.c_int, _P(_vp)]
_lib.mbci_chain3_run.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]

class mbci_funnel_t(ctypes.Structure):
    _fields_ = [("expr_raw", ctypes.c_int32), ("expr_rule1", ctypes.c_int32), ("expr_rule2", ctypes.c_int32)] + [
        (n, ctypes.c_int64) for n in ("tile_vectors", "tile_vectors_rule3", "tile_vectors_rule4", "raw",
                                      "after_rule1", "after_rule2", "after_rule3", "after_rule4")]


_lib.mbci_prune_funnel.argtypes = [ctypes.c_int64] * 4 + [ctypes.c_int32, ctypes.c_int64, _P(mbci_funnel_t)]

mbci_measure_fn = ctypes.CFUNCTYPE(ctypes.c_double, _P(mbci_plan_t), _vp)
_lib.mbci_plan_search.argtypes = [_P(mbci_chain_desc_t), _P(mbci_hw_t), _P(mbci_search_params_t), mbci_measure_fn,
                                  _vp, _P(mbci_plan_t), _P(mbci_search_result_t), _P(ctypes.c_double)]
_lib.mbci_chain_search_stats.argtypes = [_vp, _P(ctypes.c_int32), _P(ctypes.c_int32)]
for _f in ("mbci_chain_create", "mbci_chain_create_with_plan", "mbci_chain_run", "mbci_chain_run_host",
           "mbci_chain_set_trace",
           "mbci_chain_destroy", "mbci_chain_plan", "mbci_chain_describe", "mbci_plan_enumerate",
           "mbci_plan_select", "mbci_model_terms", "mbci_plan_search", "mbci_chain_search_stats",
           "mbci_chain3_create", "mbci_chain3_run", "mbci_prune_funnel",
           "mbci_chain_run_partial", "mbci_merge_partials"):
    getattr(_lib, _f).restype = _st

EXPORTED = ["mbci_chain_create", "mbci_chain_create_with_plan", "mbci_chain_run", "mbci_chain_run_host",
            "mbci_chain_destroy", "mbci_chain_plan", "mbci_chain_describe", "mbci_chain_launches_per_run",
            "mbci_chain_set_trace",
            "mbci_status_string", "mbci_last_error", "mbci_abi_version", "mbci_hw_default",
            "mbci_plan_enumerate", "mbci_plan_select", "mbci_model_terms", "mbci_plan_search",
            "mbci_chain_search_stats", "mbci_chain3_create", "mbci_chain3_run", "mbci_prune_funnel",
            "mbci_chain_run_partial", "mbci_merge_partials"]

# ---- same names as the C ABI ---------------------------------------------------------------
mbci_chain_create = _lib.mbci_chain_create
mbci_chain_create_with_plan = _lib.mbci_chain_create_with_plan
mbci_chain_run = _lib.mbci_chain_run
mbci_chain_run_host = _lib.mbci_chain_run_host
mbci_chain_destroy = _lib.mbci_chain_destroy
mbci_chain_plan = _lib.mbci_chain_plan
mbci_chain_describe = _lib.mbci_chain_describe
mbci_chain_launches_per_run = _lib.mbci_chain_launches_per_run
mbci_chain_set_trace = _lib.mbci_chain_set_trace
mbci_status_string = _lib.mbci_status_string
mbci_last_error = _lib.mbci_last_error
mbci_abi_version = _lib.mbci_abi_version
mbci_hw_default = _lib.mbci_hw_default
mbci_plan_enumerate = _lib.mbci_plan_enumerate
mbci_plan_select = _lib.mbci_plan_select
mbci_model_terms = _lib.mbci_model_terms
mbci_plan_search = _lib.mbci_plan_search
mbci_chain_search_stats = _lib.mbci_chain_search_stats
mbci_chain3_create = _lib.mbci_chain3_create
mbci_chain3_run = _lib.mbci_chain3_run
mbci_prune_funnel = _lib.mbci_prune_funnel
mbci_chain_run_partial = _lib.mbci_chain_run_partial
mbci_merge_partials = _lib.mbci_merge_partials


def plan_search(desc, measure, hw=None, N=512, n=8, eps=0.01, seed=1, max_rounds=64, model=0):
    """PAPER.md Algorithm 1 through the C ABI; `measure(plan) -> seconds` is a Python callable.
    Returns (status, best plan, result struct, per-round log [(best_est, top1_meas, best_meas)])."""
    params = mbci_search_params_t(N, n, eps, seed, max_rounds, model)
    cb = mbci_measure_fn(lambda pp, _u: float(measure(pp.contents)))
    best = mbci_plan_t()
    res = mbci_search_result_t()
    log = (ctypes.c_double * (3 * max(1, max_rounds)))()
    st = mbci_plan_search(ctypes.byref(desc), None if hw is None else ctypes.byref(hw), ctypes.byref(params), cb,
                          None, ctypes.byref(best), ctypes.byref(res), log)
    rounds = [(log[3 * i], log[3 * i + 1], log[3 * i + 2]) for i in range(res.rounds)] if st == MBCI_OK else []
    return st, best, res, rounds


class MbciError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = mbci_last_error().decode(errors="replace")
        super().__init__(f"{where}: {mbci_status_string(status).decode()} — {msg}")


def check(status, where="mbci"):
    if status != MBCI_OK:
        raise MbciError(status, where)


def make_desc(batch, M, N, K, L, dtype="bf16", op="softmax", scale=float("nan"), mask=False,
              b_layout=1, strides=None, tune=0, causal=False) -> mbci_chain_desc_t:
    d = mbci_chain_desc_t()
    d.batch, d.M, d.N, d.K, d.L = batch, M, N, K, L
    d.dtype = DTYPES[dtype] if isinstance(dtype, str) else int(dtype)
    d.op = OPS[op] if isinstance(op, str) else int(op)
    d.scale = scale
    d.mask = (MBCI_MASK_KEY_PADDING if mask else MBCI_MASK_NONE) | (MBCI_MASK_CAUSAL if causal else 0)
    d.b_layout = b_layout
    if strides:
        for k, v in strides.items():
            setattr(d, k, int(v))
    d.tune = tune
    return d


def hw_default() -> mbci_hw_t:
    hw = mbci_hw_t()
    mbci_hw_default(ctypes.byref(hw))
    return hw


def plan_enumerate(desc, hw=None, cap=512):
    arr = (mbci_plan_t * cap)()
    n = ctypes.c_int32(0)
    st = mbci_plan_enumerate(ctypes.byref(desc), ctypes.byref(hw) if hw is not None else None, arr, cap,
                             ctypes.byref(n))
    if st != MBCI_OK:
        return st, []
    return st, [arr[i] for i in range(min(cap, n.value))]


def model_terms(batch, M, N, K, L, TM, TN, TK, TH, s, hw=None):
    out = (ctypes.c_double * 5)()
    check(mbci_model_terms(batch, M, N, K, L, TM, TN, TK, TH, s,
                           ctypes.byref(hw) if hw is not None else None, out), "mbci_model_terms")
    return {"t_mem": out[0], "t_comp": out[1], "alpha": out[2], "t_estm": out[3], "n_block": out[4]}


def prune_funnel(M, N, K, H, elem_bytes=2, shm_max=232448) -> dict:
    f = mbci_funnel_t()
    check(mbci_prune_funnel(M, N, K, H, elem_bytes, shm_max, ctypes.byref(f)), "mbci_prune_funnel")
    return {name: getattr(f, name) for name, _ in f._fields_}


_TORCH_DT = None


def _torch_dtype_code(t):
    import torch
    return {torch.float32: MBCI_F32, torch.float16: MBCI_F16, torch.bfloat16: MBCI_BF16}[t]


def merge_partials(E_parts, lse_parts, E, op="softmax", stream=None):
    """E_parts [R, batch, M, L], lse_parts [R, batch, M] (fp32), E [batch, M, L]: torch tensors on one device."""
    import torch
    R, b, M, L = E_parts.shape
    s = stream if stream is not None else torch.cuda.current_stream(E.device)
    check(mbci_merge_partials(R, E_parts.data_ptr(), lse_parts.data_ptr() if lse_parts is not None else None,
                              E.data_ptr(), b, M, L, _torch_dtype_code(E.dtype),
                              OPS[op] if isinstance(op, str) else int(op), s.cuda_stream), "mbci_merge_partials")


class Chain:
    """Handle wrapper: create once per shape, run many times (torch tensors on the device)."""

    def __init__(self, batch, M, N, K, L, dtype="bf16", op="softmax", scale=float("nan"), mask=False,
                 b_layout=1, device=0, strides=None, tune=0, plan=None, causal=False):
        self.desc = make_desc(batch, M, N, K, L, dtype, op, scale, mask, b_layout, strides, tune, causal)
        self.device = device
        h = _vp()
        if plan is None:
            check(mbci_chain_create(ctypes.byref(self.desc), device, ctypes.byref(h)), "mbci_chain_create")
        else:
            check(mbci_chain_create_with_plan(ctypes.byref(self.desc), device, ctypes.byref(plan),
                                              ctypes.byref(h)), "mbci_chain_create_with_plan")
        self.h = h

    def plan(self) -> mbci_plan_t:
        p = mbci_plan_t()
        check(mbci_chain_plan(self.h, ctypes.byref(p)), "mbci_chain_plan")
        return p

    def describe(self) -> str:
        buf = ctypes.create_string_buffer(512)
        check(mbci_chain_describe(self.h, buf, 512), "mbci_chain_describe")
        return buf.value.decode()

    def set_trace(self, buf_tensor=None):
        if buf_tensor is None:
            check(mbci_chain_set_trace(self.h, None, 0), "mbci_chain_set_trace")
        else:
            check(mbci_chain_set_trace(self.h, buf_tensor.data_ptr(), buf_tensor.numel() * buf_tensor.element_size()),
                  "mbci_chain_set_trace")

    def launches_per_run(self) -> int:
        return int(mbci_chain_launches_per_run(self.h))

    def run_ptr(self, A, B, D, E, valid_len=0, stream=0):
        check(mbci_chain_run(self.h, A, B, D, E, valid_len or None, stream or None), "mbci_chain_run")

    def run(self, A, B, D, E, valid_len=None, stream=None):
        """A, B, D, E (and valid_len) are torch tensors on the handle's device."""
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.run_ptr(A.data_ptr(), B.data_ptr(), D.data_ptr(), E.data_ptr(),
                     valid_len.data_ptr() if valid_len is not None else 0, s.cuda_stream)

    def run_partial(self, A, B, D, E, lse=None, valid_len=None, key_offset=0, stream=None):
        """Split-N part over keys [key_offset, key_offset + N): E and (SOFTMAX) lse [batch, M] fp32."""
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(mbci_chain_run_partial(self.h, A.data_ptr(), B.data_ptr(), D.data_ptr(), E.data_ptr(),
                                     lse.data_ptr() if lse is not None else None,
                                     valid_len.data_ptr() if valid_len is not None else None, key_offset,
                                     s.cuda_stream), "mbci_chain_run_partial")

    def run_host(self, A, B, D, E, valid_len=None, stream=None):
        """End-to-end: host (pinned) torch tensors or numpy arrays in, host E out."""
        def ptr(x):
            if x is None:
                return None
            return x.data_ptr() if hasattr(x, "data_ptr") else x.ctypes.data
        st = stream.cuda_stream if stream is not None else None
        check(mbci_chain_run_host(self.h, ptr(A), ptr(B), ptr(D), ptr(E), ptr(valid_len), st),
              "mbci_chain_run_host")

    def close(self):
        if getattr(self, "h", None):
            mbci_chain_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def default_scale(K: int) -> float:
    return 1.0 / math.sqrt(K) if K > 0 else 1.0


class Chain3:
    """Three-contraction chain E3 = op2(op(A·B)·D)·F (mbci_chain3_*); torch tensors on the device."""

    def __init__(self, batch, M, N, K, L, H, dtype="bf16", op="softmax", scale=float("nan"), op2="none",
                 scale2=float("nan"), mask=False, causal=False, b_layout=1, device=0):
        d = mbci_chain3_desc_t()
        d.batch, d.M, d.N, d.K, d.L, d.H = batch, M, N, K, L, H
        d.dtype = DTYPES[dtype]
        d.op = OPS[op]
        d.scale = scale
        d.mask = (MBCI_MASK_KEY_PADDING if mask else 0) | (MBCI_MASK_CAUSAL if causal else 0)
        d.b_layout = b_layout
        d.op2 = OPS[op2]
        d.scale2 = scale2
        self.desc = d
        h = _vp()
        check(mbci_chain3_create(ctypes.byref(d), device, ctypes.byref(h)), "mbci_chain3_create")
        self.h = h

    def run(self, A, B, D, F, E, valid_len=None, stream=None):
        import torch
        st = (stream or torch.cuda.current_stream()).cuda_stream
        vl = None if valid_len is None else valid_len.data_ptr()
        check(mbci_chain3_run(self.h, A.data_ptr(), B.data_ptr(), D.data_ptr(), F.data_ptr(), E.data_ptr(), vl, st),
              "mbci_chain3_run")

    def plan(self):
        p = mbci_plan_t()
        check(mbci_chain_plan(self.h, ctypes.byref(p)), "mbci_chain_plan")
        return p

    def close(self):
        if getattr(self, "h", None):
            mbci_chain_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
