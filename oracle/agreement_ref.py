"""Agreement metrics, straight-line reference (TEST INFRASTRUCTURE ONLY: used by tests/ to pin
paper_2602_21144_b200/agreement.py; shares no code with it).

PAPER.md:591-610 (§5.4, Table 1): Top-1 token match, Top-5 overlap (unordered), Top-5 exact
ordered match, comparing the quantised run's next-token logits with the unquantised run's.
SPEC.md:473-487 fixes the forms: top1 = fraction of positions whose argmax agrees;
top5_unordered = mean over positions of |top5(ref) ∩ top5(test)| / 5; top5_ordered = fraction of
positions whose ordered top-5 lists are identical; ties broken to the lowest token index."""
from __future__ import annotations


def _ranked(row, k):
    # selection by repeated maximum; a later index replaces the current best only if strictly larger
    taken = set()
    out = []
    for _ in range(k):
        best = None
        for i, v in enumerate(row):
            if i in taken:
                continue
            if best is None or v > row[best]:
                best = i
        taken.add(best)
        out.append(best)
    return out


def agreement(ref, test, k=5):
    assert len(ref) == len(test)
    n = len(ref)
    t1 = un = od = 0.0
    for r, t in zip(ref, test):
        a = _ranked(list(r), k)
        b = _ranked(list(t), k)
        t1 += a[0] == b[0]
        un += len(set(a) & set(b)) / k
        od += a == b
    return t1 / n, un / n, od / n
