"""Agreement metrics between two logit streams (§5.4, Table 1: "Top-1 (argmax)",
"Top-5 overlap (Unordered)", "Top-5 (Ordered)"; SPEC.md:473-487 topk_agreement).  Host-side
evaluation of the quantised-all-reduce arms; not part of the mixer hot path.

Ties inside one logit vector are broken toward the lowest token index, the same rule as greedy
decoding."""
from __future__ import annotations

import numpy as np


def topk_ordered(logits, k):
    """[T, V] -> [T, k] token ids by descending logit, ties to the lowest index (stable sort)."""
    logits = np.asarray(logits)
    return np.argsort(-logits, axis=-1, kind="stable")[..., :k]


def topk_agreement(ref_logits, test_logits, k=5):
    """Returns dict(top1, topk_unordered, topk_ordered) averaged over positions."""
    ref_logits = np.asarray(ref_logits)
    test_logits = np.asarray(test_logits)
    if ref_logits.shape != test_logits.shape or ref_logits.ndim != 2:
        raise ValueError(f"logit streams must be [T, vocab] of equal shape: {ref_logits.shape} vs {test_logits.shape}")
    a = topk_ordered(ref_logits, k)
    b = topk_ordered(test_logits, k)
    top1 = float(np.mean(a[:, 0] == b[:, 0]))
    inter = (a[:, :, None] == b[:, None, :]).any(-1).sum(-1)   # |A ∩ B| per position
    unordered = float(np.mean(inter / k))
    ordered = float(np.mean((a == b).all(-1)))
    return {"top1": top1, f"top{k}_unordered": unordered, f"top{k}_ordered": ordered}
