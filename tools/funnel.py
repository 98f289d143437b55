"""PAPER.md Fig. 7: the pruning funnel of the paper's search space through the C ABI
(mbci_prune_funnel, csrc/prune.cpp) for the paper's example and the BASELINE shapes, on the shared-
memory budgets of the paper's GPUs (A100 163 KB, RTX 3080 99 KB) and of B200 (227 KB)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_22169_b200 import mbci

SHAPES = [("P:261 example", 1024, 1024, 512, 512), ("C2 BERT-base", 512, 512, 64, 64),
          ("C5 long-seq", 4096, 4096, 128, 128), ("C6 ViT-base", 197, 197, 64, 64),
          ("Table II G4", 512, 512, 256, 64), ("ragged 1000x500", 1000, 1000, 500, 500)]
GPUS = [("A100", 166912), ("RTX3080", 101376), ("B200", 232448)]
print(f"{'shape':18s} {'gpu':8s} {'raw':>11s} {'R1 (expr)':>16s} {'R2 (expr)':>15s} {'R3':>8s} {'R3 drop':>8s} {'R4':>7s} {'R4 drop':>8s}")
for name, M, N, K, H in SHAPES:
    for g, shm in GPUS:
        f = mbci.prune_funnel(M, N, K, H, 2, shm)
        print(f"{name:18s} {g:8s} {f['raw']:11d} {f['after_rule1']:10d} ({f['expr_rule1']}) {f['after_rule2']:9d} ({f['expr_rule2']}) "
              f"{f['after_rule3']:8d} {1 - f['tile_vectors_rule3'] / f['tile_vectors']:8.4f} {f['after_rule4']:7d} "
              f"{1 - f['tile_vectors_rule4'] / max(1, f['tile_vectors_rule3']):8.3f}")
print("paper (Fig. 7, P:311): expressions 26 -> 5 (Rule 1) -> 3 (Rule 2); Rule 3 discards 99 %, Rule 4 40 %; 10^8 -> 10^4")
