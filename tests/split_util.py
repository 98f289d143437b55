"""Host-side helpers of the split-N tests: key-range views of seeded inputs and the
log-sum-exp combination of partial results written out from its definition (E = Σ w_r E_r / Σ w_r,
w_r = exp(lse_r − max lse)), used to check the oracle's partials against its full chain."""
import numpy as np

import mbci_inputs as gen


def slice_keys(inp, n0, n1):
    """ChainInputs over keys [n0, n1) of inp (packed copies of the B and D key ranges)."""
    B = inp.B[:, :, n0:n1] if inp.b_layout == 0 else inp.B[:, n0:n1, :]
    return gen.ChainInputs(inp.A, np.ascontiguousarray(B), np.ascontiguousarray(inp.D[:, n0:n1, :]), None,
                           inp.dtype, inp.batch, inp.M, n1 - n0, inp.K, inp.L, inp.b_layout)


def local_valid(valid_len, n0, n1):
    return None if valid_len is None else np.clip(np.asarray(valid_len) - n0, 0, n1 - n0).astype(np.int32)


def lse_combine(E_parts, lse_parts):
    """Σ_r w_r E_r / Σ_r w_r over axis 0 (float64); rows with every lse = −inf give 0."""
    lse = np.asarray(lse_parts, dtype=np.float64)
    mx = lse.max(axis=0)
    safe = np.where(np.isfinite(mx), mx, 0.0)
    w = np.where(np.isfinite(lse), np.exp(lse - safe[None]), 0.0)
    s = w.sum(axis=0)
    num = (w[..., None] * np.asarray(E_parts, dtype=np.float64)).sum(axis=0)
    return np.where(s[..., None] > 0, num / np.where(s > 0, s, 1.0)[..., None], 0.0)
