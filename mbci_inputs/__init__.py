"""Seeded synthetic inputs for the fused MBCI chain E = op(A·B)·D.

This module is the ONLY code shared by the CPU oracle (``oracle/``) and the
CUDA path (``paper_2506_22169_b200``).  It holds no arithmetic of the method:
it only draws numbers and stores them as raw bits.

Recipe (DESIGN.md §3 "Input recipe"; SURVEY.md §8(d) "Seeds"):
  element ``i`` of tensor ``t`` under seed ``s`` is
  ``x = splitmix64(s ^ (t << 56) ^ i)``; the high 32 bits give ``u1`` and the
  low 32 bits ``u2`` (both mapped to (0,1)); Box–Muller gives
  ``z = sqrt(-2 ln u1) * cos(2π u2)``; the value is ``sigma * z`` rounded
  RN-even to the storage dtype (fp32: numpy float64→float32; fp16: numpy
  float64→float16; bf16: float64→float32 (RN) then float32→bf16 RN-even on
  the bit pattern).  Because the generator is counter-based, any batch slice
  (a multi-GPU shard) is generated independently and bit-identically to the
  same rows of the full tensor.

Integer variant (``kind="int"``): ``(x >> 32) % (2*r+1) - r`` — small integers
that every dtype holds exactly.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "DTYPES", "splitmix64", "normal_bits", "int_bits", "bits_to_f64_numpy",
    "valid_lengths", "ChainInputs", "make_chain_inputs", "dtype_size",
]

DTYPES = {"f32": 4, "f16": 2, "bf16": 2}
TENSOR_IDS = {"A": 1, "B": 2, "D": 3, "VL": 4}

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def dtype_size(dtype: str) -> int:
    return DTYPES[dtype]


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Steele/Lea/Flood splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def _counters(seed: int, tensor: str, start: int, count: int) -> np.ndarray:
    base = np.uint64((seed & 0xFFFFFFFFFFFFFFFF) ^ ((TENSOR_IDS[tensor] & 0xFF) << 56))
    idx = np.arange(start, start + count, dtype=np.uint64)
    return splitmix64(idx ^ base)


def _f64_to_storage(v: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "f32":
        return v.astype(np.float32).view(np.uint32)
    if dtype == "f16":
        return v.astype(np.float16).view(np.uint16)
    if dtype == "bf16":
        f = v.astype(np.float32).view(np.uint32).astype(np.uint64)
        # RN-even on the low 16 bits (inputs here are finite, never NaN)
        rounded = (f + np.uint64(0x7FFF) + ((f >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
        return rounded.astype(np.uint16)
    raise ValueError(dtype)


def normal_bits(seed: int, tensor: str, start: int, count: int, dtype: str,
                sigma: float = 1.0, chunk: int = 1 << 24) -> np.ndarray:
    """``count`` N(0, sigma^2) draws (elements start..start+count-1 of tensor) as raw storage bits."""
    out = np.empty(count, dtype=np.uint32 if dtype == "f32" else np.uint16)

    def fill(c0):
        n = min(chunk, count - c0)
        x = _counters(seed, tensor, start + c0, n)
        u1 = ((x >> np.uint64(32)).astype(np.float64) + 0.5) * (1.0 / 4294967296.0)
        u2 = ((x & np.uint64(0xFFFFFFFF)).astype(np.float64) + 0.5) * (1.0 / 4294967296.0)
        z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
        out[c0:c0 + n] = _f64_to_storage(sigma * z, dtype)

    starts = range(0, count, chunk)
    if len(starts) > 1:   # disjoint chunks; numpy releases the GIL, so host threads help at C5 sizes
        with ThreadPoolExecutor(max_workers=min(len(starts), os.cpu_count() or 1, 32)) as ex:
            list(ex.map(fill, starts))
    else:
        for c0 in starts:
            fill(c0)
    return out


def int_bits(seed: int, tensor: str, start: int, count: int, dtype: str, r: int = 2) -> np.ndarray:
    """Small integers in [-r, r] (exact in every dtype) as raw storage bits."""
    x = _counters(seed, tensor, start, count)
    v = ((x >> np.uint64(32)) % np.uint64(2 * r + 1)).astype(np.int64) - r
    return _f64_to_storage(v.astype(np.float64), dtype)


def bits_to_f64_numpy(bits: np.ndarray, dtype: str) -> np.ndarray:
    """Library decode (numpy) of storage bits.  Used by tests as an independent
    check of the oracle's own bit decoder, and by the harness for display."""
    if dtype == "f32":
        return bits.view(np.float32).astype(np.float64)
    if dtype == "f16":
        return bits.view(np.float16).astype(np.float64)
    if dtype == "bf16":
        return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
    raise ValueError(dtype)


def valid_lengths(seed: int, batch: int, lo: int, hi: int, start: int = 0) -> np.ndarray:
    """Per-batch key-padding lengths uniform in [lo, hi] (inclusive)."""
    x = _counters(seed, "VL", start, batch)
    span = np.uint64(hi - lo + 1)
    return ((x >> np.uint64(32)) % span).astype(np.int64).astype(np.int32) + np.int32(lo)


class ChainInputs:
    """Raw-bit inputs of one chain problem (packed, row-major)."""

    def __init__(self, A, B, D, valid_len, dtype, batch, M, N, K, L, b_layout):
        self.A, self.B, self.D = A, B, D
        self.valid_len = valid_len
        self.dtype = dtype
        self.batch, self.M, self.N, self.K, self.L = batch, M, N, K, L
        self.b_layout = b_layout

    def shapes(self):
        B_shape = (self.batch, self.K, self.N) if self.b_layout == 0 else (self.batch, self.N, self.K)
        return (self.batch, self.M, self.K), B_shape, (self.batch, self.N, self.L)


def make_chain_inputs(seed: int, dtype: str, batch: int, M: int, N: int, K: int, L: int,
                      b_layout: int = 1, kind: str = "normal", sigmas=(1.0, 1.0, 1.0),
                      batch_start: int = 0, valid_len_range=None) -> ChainInputs:
    """Inputs for batch rows ``batch_start .. batch_start+batch-1`` of a problem.

    ``kind``: "normal" (N(0, sigma^2) per tensor, sigmas = (sA, sB, sD)) or "int".
    Element indices are global (batch_start included) so a shard is bit-identical
    to the same rows of the unsharded tensor.
    """
    nA, nB, nD = M * K, K * N, N * L
    if kind == "normal":
        A = normal_bits(seed, "A", batch_start * nA, batch * nA, dtype, sigmas[0])
        B = normal_bits(seed, "B", batch_start * nB, batch * nB, dtype, sigmas[1])
        D = normal_bits(seed, "D", batch_start * nD, batch * nD, dtype, sigmas[2])
    elif kind == "int":
        A = int_bits(seed, "A", batch_start * nA, batch * nA, dtype)
        B = int_bits(seed, "B", batch_start * nB, batch * nB, dtype)
        D = int_bits(seed, "D", batch_start * nD, batch * nD, dtype)
    else:
        raise ValueError(kind)
    vl = None
    if valid_len_range is not None:
        vl = valid_lengths(seed, batch, valid_len_range[0], valid_len_range[1], start=batch_start)
    B_shape = (batch, K, N) if b_layout == 0 else (batch, N, K)
    return ChainInputs(A.reshape(batch, M, K), B.reshape(B_shape), D.reshape(batch, N, L),
                       vl, dtype, batch, M, N, K, L, b_layout)
