"""Shared helpers for the -m gpu tests: move generator bits to the device, run the chain
through the C ABI, read E back as float64 and as raw bits."""
import numpy as np
import torch

import mbci_inputs as gen

TORCH_DT = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}


def to_dev(bits, dtype, dev="cuda"):
    if dtype == "f32":
        t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int32))
    else:
        t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16))
    return t.to(dev).view(TORCH_DT[dtype])


def e_bits(E):
    """Raw storage bits of a device E tensor as a numpy uint array."""
    if E.dtype == torch.float32:
        return E.cpu().view(torch.int32).numpy().view(np.uint32)
    return E.cpu().view(torch.int16).numpy().view(np.uint16)


def e_f64(E, dtype):
    return gen.bits_to_f64_numpy(e_bits(E), dtype)


def run_chain(mbci, inp, op, scale, valid_len=None, plan=None, E=None, tune=0, causal=False):
    """Create a handle for inp's shape, run once, return (E tensor, Chain)."""
    dev = torch.device("cuda", 0)
    ch = mbci.Chain(inp.batch, inp.M, inp.N, inp.K, inp.L, inp.dtype, op, scale,
                    mask=valid_len is not None, b_layout=inp.b_layout, device=0, plan=plan, tune=tune,
                    causal=causal)
    A = to_dev(inp.A, inp.dtype)
    B = to_dev(inp.B, inp.dtype)
    D = to_dev(inp.D, inp.dtype)
    if E is None:
        E = torch.full((inp.batch, inp.M, inp.L), float("nan"), dtype=TORCH_DT[inp.dtype], device=dev)
    vl = None if valid_len is None else torch.from_numpy(np.asarray(valid_len, dtype=np.int32)).to(dev)
    ch.run(A, B, D, E, vl)
    torch.cuda.synchronize()
    return E, ch


def rn_bits(E_f64, dtype):
    """RN-even storage bits of float64 values (numpy) — for bitwise comparisons."""
    return gen._f64_to_storage(np.asarray(E_f64, dtype=np.float64).ravel(), dtype).reshape(np.shape(E_f64))
