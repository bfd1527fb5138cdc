"""Confusion counts, pinned to the reference's
evaluate.accumulate (evaluate.py:87-106) on seeded masks and ground truth
(tests/golden/confusion_vectors.npz, made by tests/golden/make_golden.py)."""

from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

import paper_1302_2073_b200 as pkg

GOLD = Path(__file__).resolve().parent / "golden" / "confusion_vectors.npz"


def _cases():
    z = np.load(GOLD)
    i = 0
    while f"dims{i}" in z:
        yield z[f"dims{i}"], z[f"mask{i}"], z[f"gt{i}"], z[f"counts{i}"]
        i += 1


def test_golden_counts_are_consistent():
    for (w, h), m, g, c in _cases():
        scored = np.sum((g != 85) & (g != 170))
        assert int(c.sum()) == int(scored)


@pytest.mark.gpu
def test_device_counts_match_reference():
    import torch
    from paper_1302_2073_b200.scoring import ConfusionCounts, accumulate, accumulate_device

    for (w, h), m, g, c in _cases():
        got = accumulate(ConfusionCounts(), pkg.SegmentationMask(int(w), int(h), m),
                         SimpleNamespace(width=int(w), height=int(h), labels=g))
        assert (got.tp, got.fp, got.tn, got.fn) == tuple(int(v) for v in c)
    # batched, accumulating twice over the same frames doubles the counts
    cases = list(_cases())
    (w, h), m, g, c = cases[0]
    S = 3
    masks = torch.from_numpy(np.tile(m, S)).cuda()
    truths = torch.from_numpy(np.tile(g, (S, 1))).cuda()
    counts = torch.zeros((S, 4), dtype=torch.int64, device="cuda")
    accumulate_device(counts, masks, truths)
    accumulate_device(counts, masks, truths)
    np.testing.assert_array_equal(counts.cpu().numpy(), np.tile(2 * c, (S, 1)))
