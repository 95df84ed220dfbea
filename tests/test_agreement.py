"""Agreement metrics (Table 1): the harness' vectorised
implementation against a straight-line oracle and SPEC's constructed examples."""
import numpy as np
import pytest

from oracle import agreement_ref as R
from paper_2602_21144_b200.agreement import topk_agreement


def test_identical_streams():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((20, 50))
    m = topk_agreement(x, x)
    assert (m["top1"], m["top5_unordered"], m["top5_ordered"]) == (1.0, 1.0, 1.0)


def test_swapped_top2():
    """top-2 swapped at every position -> top1 0, unordered 1, ordered 0."""
    rng = np.random.default_rng(1)
    x = rng.standard_normal((16, 40))
    y = x.copy()
    o = np.argsort(-x, axis=1)
    for t in range(16):
        i, j = o[t, 0], o[t, 1]
        y[t, i], y[t, j] = x[t, j], x[t, i]
    m = topk_agreement(x, y)
    assert (m["top1"], m["top5_unordered"], m["top5_ordered"]) == (0.0, 1.0, 0.0)


def test_ties_lowest_index():
    x = np.array([[1.0, 3.0, 3.0, 0.0, 3.0, 2.0, 2.0]])
    y = np.array([[0.0, 3.0, 3.0, 1.0, 3.0, 2.0, 2.0]])
    m = topk_agreement(x, y, k=5)
    # ranked: x -> [1, 2, 4, 5, 6]; y -> [1, 2, 4, 5, 6]
    assert m["top5_ordered"] == 1.0
    assert R.agreement(x, y, 5) == (1.0, 1.0, 1.0)


@pytest.mark.parametrize("scale", [0.0, 0.05, 0.3, 1.0])
def test_matches_straight_line_reference(scale):
    """a seeded Gaussian perturbation; all three metrics equal an independent
    straight-line recomputation (including ties from a coarse grid)."""
    rng = np.random.default_rng(7)
    x = np.round(rng.standard_normal((40, 30)) * 4) / 4          # coarse grid: many ties
    y = x + scale * rng.standard_normal(x.shape)
    m = topk_agreement(x, y)
    t1, un, od = R.agreement(x, y, 5)
    assert m["top1"] == pytest.approx(t1, abs=1e-12)
    assert m["top5_unordered"] == pytest.approx(un, abs=1e-12)
    assert m["top5_ordered"] == pytest.approx(od, abs=1e-12)
    assert m["top5_unordered"] >= m["top5_ordered"]


def test_shape_mismatch_raises():
    with pytest.raises(ValueError):
        topk_agreement(np.zeros((3, 5)), np.zeros((4, 5)))
