"""Paper formulas for the tile selector, written from PAPER.md (test oracle only).

Every function restates one passage; no function is shared with the CUDA
library's selector (paper_2506_22169_b200/csrc/selector.cpp), which
re-implements the same formulas in C++ and is checked against these.

  phi_printed     PAPER.md:119 (§II-A): phi = 2 T_M T_N K / (2 T_M T_N + T_M K + T_N K)
  phi_text        the reading that reproduces PAPER.md:78 (§I, "from 227 to 2") with
                  the 256-tile of Fig. 2: output counted once
  fused_intensity (M+N)(K+L)s bytes vs 2MN(K+L) FLOPs (SURVEY §0 finding 2)
  is_memory_bound PAPER.md:119: "transitions to a memory-bound state when phi < P/W"
  n_deep / n_flat PAPER.md:199-200 (§III-A): x! deep expressions, 2 flat ones
  space_size      PAPER.md:261 (§III-C): (24+2) x ceil(1024/16)^2 x ceil(512/16)^2
  tile_options    PAPER.md:203: multiples of 16 up to the (padded) dimension
  rule3_reject    PAPER.md:288 (Rule 3)
  shm_estm        PAPER.md:307-309 (Eq. 1); Rule 4 PAPER.md:290 (> 1.2 Shm_max)
  t_mem/t_comp/alpha/t_estm   PAPER.md:324-339 (Eqs. 2-5)
  chain_schedule  the flat chain schedule mh(n(k(L_A,L_B,C_C),L_D,C_E),S_E)
                   with dead-loop elimination
"""
from __future__ import annotations

import itertools
import math


# ---- §II-A ---------------------------------------------------------------
def phi_printed(TM: float, TN: float, K: float) -> float:
    return 2.0 * TM * TN * K / (2.0 * TM * TN + TM * K + TN * K)


def phi_text(TM: float, TN: float, K: float) -> float:
    return 2.0 * TM * TN * K / (TM * TN + TM * K + TN * K)


def fused_intensity(M, N, K, L, s) -> float:
    """FLOP per HBM byte of the fused chain: 2MN(K+L) / ((M K + K N + N L + M L) s)."""
    return 2.0 * M * N * (K + L) / ((M * K + K * N + N * L + M * L) * s)


def is_memory_bound(phi: float, P: float, W: float) -> bool:
    return phi < P / W


# ---- §III-A / §III-C -------------------------------------------------------
def deep_expressions(axes=("m", "n", "k", "h")):
    return ["".join(p) for p in itertools.permutations(axes)]


def flat_expressions():
    # "two flat tiling expressions exist: mn(k,h) and nm(k,h)"
    return ["mn(k,h)", "nm(k,h)"]


def tile_options(dim: int, min_tile: int = 16):
    return [min_tile * i for i in range(1, math.ceil(dim / min_tile) + 1)]


def space_size(M: int, N: int, K: int, H: int, min_tile: int = 16) -> int:
    n_expr = len(deep_expressions()) + len(flat_expressions())
    return n_expr * math.ceil(M / min_tile) * math.ceil(N / min_tile) * \
        math.ceil(K / min_tile) * math.ceil(H / min_tile)


def rule3_reject(size: int, tile: int) -> bool:
    """Rule 3: reject padded tiles on power-of-2 dims; otherwise padding ratio must stay < 0.05."""
    if size % tile == 0:
        return False
    if size & (size - 1) == 0:
        return True
    pad = math.ceil(size / tile) * tile - size
    return pad / size >= 0.05


def shm_estm(tiles) -> float:
    """Eq. (1): sum over in-block tiles X_i in R^{L_i x L_j} of T_{L_i} x T_{L_j} (elements;
    multiply by the element size for bytes)."""
    return float(sum(a * b for a, b in tiles))


def rule4_reject(shm_bytes: float, shm_max: float) -> bool:
    return shm_bytes > 1.2 * shm_max


# ---- §IV-A Eqs. (2)-(5) ----------------------------------------------------
def t_mem(mem_statements, W: float) -> float:
    """Eq. (3): sum over Load/Store statements of TS x prod(trip counts) / W.
    mem_statements: iterable of (TS_bytes, [loop extents of Lp_set])."""
    return sum(ts * math.prod(lp) for ts, lp in mem_statements) / W


def t_comp(compute_statements, P: float) -> float:
    """Eq. (4): sum over Compute statements of Fp x prod(trip counts) / P."""
    return sum(fp * math.prod(lp) for fp, lp in compute_statements) / P


def alpha(n_block: int, n_sm: int) -> float:
    """Eq. (5): (N_block + N_SM) / N_block."""
    return (n_block + n_sm) / n_block


def t_estm(tm: float, tc: float, a: float) -> float:
    """Eq. (2): (t_mem + t_comp) x alpha."""
    return (tm + tc) * a


def chain_schedule(batch, M, N, K, L, TM, TN, TK, TH, s):
    """Statements of the flat chain schedule mh(n(k(L_A,L_B,C_C),L_D,C_E),S_E).

    Loops (extents): batch b, m = ceil(M/TM), h = ceil(L/TH), n = ceil(N/TN),
    k = ceil(K/TK).  Placement follows PAPER.md:230-253: each memory statement
    sits in the scope of its innermost live related loop; a loop of extent 1 is
    dead and removed, so its statements move outward.
      L_A  related {m,k}  -> scope m,h,n,k while k is live; m only when k is dead
      L_B  related {k,n}  -> scope m,h,n,k
      C_C  Fp = 2 TM TN TK, scope m,h,n,k
      L_D  related {n,h}  -> scope m,h,n
      C_E  Fp = 2 TM TN TH, scope m,h,n
      S_E  related {m,h}  -> scope m,h (hoisted out of n: PAPER.md:232-233)
    Returns (mem_statements, compute_statements, n_block) for Eqs. (3)-(5);
    blockIdx binds m and h (Rule 1) and the batch.
    """
    b = batch
    lm, lh, ln, lk = (math.ceil(M / TM), math.ceil(L / TH), math.ceil(N / TN), math.ceil(K / TK))
    if lk == 1:
        la = [b, lm]                 # dead k: L_A moves to m scope ("a factor of hn")
    else:
        la = [b, lm, lh, ln, lk]
    mem = [
        (TM * TK * s, la),                    # L_A
        (TK * TN * s, [b, lm, lh, ln, lk]),   # L_B
        (TN * TH * s, [b, lm, lh, ln]),       # L_D
        (TM * TH * s, [b, lm, lh]),           # S_E
    ]
    comp = [
        (2.0 * TM * TN * TK, [b, lm, lh, ln, lk]),  # C_C
        (2.0 * TM * TN * TH, [b, lm, lh, ln]),      # C_E
    ]
    return mem, comp, b * lm * lh


def chain_estimate(batch, M, N, K, L, TM, TN, TK, TH, s, W, P, n_sm):
    mem, comp, nb = chain_schedule(batch, M, N, K, L, TM, TN, TK, TH, s)
    tm, tc, a = t_mem(mem, W), t_comp(comp, P), alpha(nb, n_sm)
    return {"t_mem": tm, "t_comp": tc, "alpha": a, "t_estm": t_estm(tm, tc, a), "n_block": nb}


# ---- §III-C pruning (Rules 1-4) and the Fig. 7 funnel ----------------------
# PAPER.md:283-312.  Readings (R21): Rule 1 binds the spatial loops of the final output
# (m and h of E) to blockIdx and deletes them wherever they appear (the paper's own example
# "both mhnk and mnkh yield the same sub-tiling expression nk"); Rule 2 rejects a class
# whose producer reduction k encloses the producer's spatial loop n ("reduced loop positioned
# outside the spatial loops", Fig. 6(b): `kn`); Rule 3 as rule3_reject on every axis;
# Rule 4 with Eq. (1) over the five in-block tiles A (TM x TK), B (TK x TN), C (TM x TN),
# D (TN x TH), E (TM x TH) times the element size, rejected when > 1.2 Shm_max.
def sub_tiling_expression(expr: str, bound: str = "mh") -> str:
    """Rule 1 key: delete the blockIdx-bound loops; an emptied or one-child Seq collapses."""
    out = "".join(c for c in expr if c not in bound)
    out = out.replace("(,", "(").replace(",)", ")").replace("()", "")
    if "(" in out and "," not in out:   # n(k) stays a Seq of one child: print as n(k)
        pass
    return out


def rule2_reject(key: str) -> bool:
    """the producer C's reduction loop k outside its spatial loop n caches many C tiles."""
    return "k" in key and "n" in key and key.index("k") < key.index("n")


def prune_funnel(M: int, N: int, K: int, H: int, elem_bytes: int, shm_max: float):
    """Fig. 7: candidate counts (expression x tile vector) after each rule."""
    import numpy as np
    exprs = deep_expressions() + flat_expressions()
    keys = []
    for e in exprs:   # first writer wins (canonical order: deep permutations, then flat)
        k = sub_tiling_expression(e)
        if k not in keys:
            keys.append(k)
    kept = [k for k in keys if not rule2_reject(k)]
    opts = [tile_options(d) for d in (M, N, K, H)]
    v_raw = math.prod(len(o) for o in opts)
    surv = [np.array([t for t in o if not rule3_reject(d, t)], dtype=np.float64)
            for o, d in zip(opts, (M, N, K, H))]
    v3 = math.prod(len(s) for s in surv)
    TM, TN, TK, TH = np.meshgrid(*surv, indexing="ij")
    shm = (TM * TK + TK * TN + TM * TN + TN * TH + TM * TH) * elem_bytes   # Eq. (1)
    v4 = int(np.count_nonzero(~(shm > 1.2 * shm_max)))
    return {
        "expr_raw": len(exprs), "expr_rule1": len(keys), "expr_rule2": len(kept), "keys": keys,
        "tile_vectors": v_raw, "tile_vectors_rule3": v3, "tile_vectors_rule4": v4,
        "raw": len(exprs) * v_raw, "after_rule1": len(keys) * v_raw,
        "after_rule2": len(kept) * v_raw, "after_rule3": len(kept) * v3,
        "after_rule4": len(kept) * v4,
    }
