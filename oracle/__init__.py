"""CPU oracle for the fused MBCI chain E = op(A·B)·D (MCFuser, arXiv 2506.22169).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2506_22169_b200``) never imports it, and
it never imports the product path; the two share only ``mbci_inputs`` (seeded
input bits, no arithmetic of the method).

Contents
  * ``chain``      — the plain unfused chain in fp64 (``mbci_oracle.c``; see its
                     header for the PAPER.md passages it follows).
  * ``decode``     — the oracle's own IEEE fp16 / bf16 / fp32 bit decoders.
  * ``model``      — §II-A φ, §III-A search-space counts, §III-C Rules 3/4 +
                     Eq. (1), §IV-A Eqs. (2)-(5) (pure Python, written from the text).

Pins (tests/test_oracle_pins.py) tie each function to something other than
itself: SDPA from torch (a library routine), associativity with exact integer
inputs, D = I, zero-K / scale = 0 / single-key closed forms, row sums, shift
invariance, numpy's fp16 conversion, and the paper's printed numbers.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import model  # noqa: F401  (re-export)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mbci_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_LIB = None

DTYPE_CODE = {"f32": 0, "f16": 1, "bf16": 2}
OP_CODE = {"none": 0, "scale": 1, "softmax": 2, "relu": 3, "gelu": 4}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, -O2, OpenMP; no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _LIB_PATH, _SRC, "-lm"])
    return _LIB_PATH


def lib():
    global _LIB
    if _LIB is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, vp, dp = ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p
        L.oracle_chain.argtypes = [vp, vp, vp, dp, ctypes.c_int, i64, i64, i64, i64, i64,
                                   ctypes.c_int, ctypes.c_double, ctypes.c_int, vp, vp, i64,
                                   ctypes.c_int, dp]
        L.oracle_chain.restype = ctypes.c_int
        L.oracle_chain_ex.argtypes = [vp, vp, vp, dp, ctypes.c_int, i64, i64, i64, i64, i64,
                                      ctypes.c_int, ctypes.c_double, ctypes.c_int, vp, ctypes.c_int, vp, i64,
                                      ctypes.c_int, dp]
        L.oracle_chain_ex.restype = ctypes.c_int
        L.oracle_chain3.argtypes = [vp, vp, vp, vp, dp, ctypes.c_int, i64, i64, i64, i64, i64, i64, ctypes.c_int,
                                    ctypes.c_double, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_double, ctypes.c_int]
        L.oracle_chain3.restype = ctypes.c_int
        L.oracle_row_lse.argtypes = [vp, vp, dp, ctypes.c_int, i64, i64, i64, i64, ctypes.c_double, ctypes.c_int,
                                     vp, ctypes.c_int]
        L.oracle_decode_array.argtypes = [vp, ctypes.c_int, i64, dp]
        L.oracle_decode_array.restype = ctypes.c_int
        L.oracle_max_threads.restype = ctypes.c_int
        for f in ("oracle_decode_f16", "oracle_decode_bf16"):
            getattr(L, f).argtypes = [ctypes.c_uint16]
            getattr(L, f).restype = ctypes.c_double
        L.oracle_decode_f32.argtypes = [ctypes.c_uint32]
        L.oracle_decode_f32.restype = ctypes.c_double
        _LIB = L
    return _LIB


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def decode(bits: np.ndarray, dtype: str) -> np.ndarray:
    """Oracle bit decoder: storage bits -> float64 (exact)."""
    bits = np.ascontiguousarray(bits)
    out = np.empty(bits.shape, dtype=np.float64)
    rc = lib().oracle_decode_array(_ptr(bits), DTYPE_CODE[dtype], bits.size, _ptr(out))
    assert rc == 0
    return out


def chain(inp, op: str, scale: float = 1.0, valid_len=None, rows=None,
          nthreads: int = 0, want_cprime: bool = False, causal: bool = False):
    """fp64 E for ``inp`` (an ``mbci_inputs.ChainInputs``).

    rows: None (all rows; E is [batch, M, L]) or an int64 array of (β, m) pairs
    (E is [len(rows), L]).  valid_len: None or int32[batch] (softmax key padding).
    causal: softmax sees key n from row m only if n <= m (R18).
    Returns E, or (E, C') when want_cprime.
    """
    A = np.ascontiguousarray(inp.A)
    B = np.ascontiguousarray(inp.B)
    D = np.ascontiguousarray(inp.D)
    vl = None if valid_len is None else np.ascontiguousarray(valid_len, dtype=np.int32)
    if rows is None:
        nrows = inp.batch * inp.M
        E = np.empty((inp.batch, inp.M, inp.L), dtype=np.float64)
        rr = None
    else:
        rr = np.ascontiguousarray(np.asarray(rows, dtype=np.int64).reshape(-1, 2))
        nrows = rr.shape[0]
        E = np.empty((nrows, inp.L), dtype=np.float64)
    Cp = np.empty((nrows, inp.N), dtype=np.float64) if want_cprime else None
    rc = lib().oracle_chain_ex(_ptr(A), _ptr(B), _ptr(D), _ptr(E), DTYPE_CODE[inp.dtype],
                               inp.batch, inp.M, inp.N, inp.K, inp.L, OP_CODE[op], float(scale),
                               inp.b_layout, _ptr(vl), 1 if causal else 0, _ptr(rr),
                               0 if rr is None else nrows, int(nthreads), _ptr(Cp))
    if rc != 0:
        raise ValueError("oracle_chain rejected its arguments")
    return (E, Cp) if want_cprime else E


def row_lse(inp, scale: float, valid_len=None, nthreads: int = 0) -> np.ndarray:
    """fp64 [batch, M]: ln sum_{n < valid} exp(scale * (A.B)[m, n]) (-inf without a valid key) — the
    statistic of a split-N partial."""
    A = np.ascontiguousarray(inp.A)
    B = np.ascontiguousarray(inp.B)
    vl = None if valid_len is None else np.ascontiguousarray(valid_len, dtype=np.int32)
    out = np.empty((inp.batch, inp.M), dtype=np.float64)
    rc = lib().oracle_row_lse(_ptr(A), _ptr(B), _ptr(out), DTYPE_CODE[inp.dtype], inp.batch, inp.M, inp.N, inp.K,
                              float(scale), inp.b_layout, _ptr(vl), int(nthreads))
    if rc != 0:
        raise ValueError("oracle_row_lse rejected its arguments")
    return out


def chain3(inp, F, H: int, op: str, scale: float, op2: str, scale2: float = 1.0, valid_len=None,
           causal: bool = False, nthreads: int = 0):
    """fp64 E3 [batch, M, H] = op2(op(A·B)·D) · F for ``inp`` and F (storage bits [batch, L, H])."""
    A = np.ascontiguousarray(inp.A)
    B = np.ascontiguousarray(inp.B)
    D = np.ascontiguousarray(inp.D)
    Fb = np.ascontiguousarray(F)
    vl = None if valid_len is None else np.ascontiguousarray(valid_len, dtype=np.int32)
    E = np.empty((inp.batch, inp.M, H), dtype=np.float64)
    rc = lib().oracle_chain3(_ptr(A), _ptr(B), _ptr(D), _ptr(Fb), _ptr(E), DTYPE_CODE[inp.dtype], inp.batch,
                             inp.M, inp.N, inp.K, inp.L, H, OP_CODE[op], float(scale), inp.b_layout, _ptr(vl),
                             1 if causal else 0, OP_CODE[op2], float(scale2), int(nthreads))
    if rc != 0:
        raise ValueError("oracle_chain3 rejected its arguments")
    return E


def row_max_error(E_gpu: np.ndarray, E_ref: np.ndarray) -> float:
    """SURVEY §8(c) comparator: max over rows of max_l |E_gpu - E_ref| / max_l |E_ref|
    (absolute error for a row whose reference is all zero)."""
    Eg = np.asarray(E_gpu, dtype=np.float64).reshape(-1, E_ref.shape[-1])
    Er = np.asarray(E_ref, dtype=np.float64).reshape(-1, E_ref.shape[-1])
    if Er.size == 0:
        return 0.0
    diff = np.abs(Eg - Er).max(axis=1)
    den = np.abs(Er).max(axis=1)
    err = np.where(den > 0, diff / np.where(den > 0, den, 1.0), diff)
    return float(err.max())
