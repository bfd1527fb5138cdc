"""Resampling shell: bilinear frame resampling and
nearest mask upsampling (reference pipeline.py:164-193, 245-258), pinned to
vectors produced by the reference itself (tests/golden/resample_vectors.npz).

CPU: the oracle restatement equals the reference bit for bit.  GPU: the
device kernels equal the reference bit for bit (fp64, no FMA contraction), and
StreamTracker.push resamples off-resolution frames as the reference does.
"""

from pathlib import Path

import numpy as np
import pytest

import paper_1302_2073_b200 as pkg
from oracle import prost_oracle as orc

GOLD = Path(__file__).resolve().parent / "golden" / "resample_vectors.npz"


def _cases():
    z = np.load(GOLD)
    i = 0
    while f"dims{i}" in z:
        yield z[f"dims{i}"], z[f"in{i}"], z[f"out{i}"], z[f"lab{i}"], z[f"up{i}"]
        i += 1


def test_oracle_resample_matches_reference():
    for (c, w, h, ow, oh), x, out, lab, up in _cases():
        np.testing.assert_array_equal(orc.resample_planes(x, c, w, h, ow, oh), out)
        np.testing.assert_array_equal(orc.upsample_labels(lab, w, h, ow, oh), up)


@pytest.mark.gpu
def test_device_resample_matches_reference():
    from paper_1302_2073_b200.resample import resample, upsample_mask

    for (c, w, h, ow, oh), x, out, lab, up in _cases():
        got = resample(pkg.FrameBuffer(int(w), int(h), int(c), x), int(ow), int(oh))
        np.testing.assert_array_equal(got.data, out)
        m = upsample_mask(pkg.SegmentationMask(int(w), int(h), lab), int(ow), int(oh))
        np.testing.assert_array_equal(m.labels, up)


@pytest.mark.gpu
def test_stream_tracker_resamples_off_resolution_frames():
    """jobs.py:181-184: a 40x30 camera into a 32x24 model, against the oracle
    fed the reference-resampled frames (fp64: identical masks)."""
    from paper_1302_2073_b200.synth import SceneSpec, SceneStream

    raw = SceneStream(SceneSpec(width=40, height=30, channels=1, rank=3, seed=8)).next_frames(10)
    cfg = pkg.RunConfig(subspace_dim=4, p=0.5, mu=1e-4, cg_max_iters=2, target_width=32,
                        target_height=24, grayscale=True, i_init=4, seed=1)
    tr = pkg.StreamTracker(cfg, precision="fp64")
    prm = cfg.params(4)
    ref = orc.PipelineOracle(32, 24, 1, orc.OracleParams(
        k=4, p=0.5, mu=1e-4, delta=prm.delta, omega=prm.omega, t_init=prm.t_init,
        t_min=prm.t_min, tau=prm.tau, max_iters=2), i_init=4, seed=1)
    for v in raw:
        a = tr.push(pkg.FrameBuffer(40, 30, 1, v))
        b = ref.push(orc.resample_planes(v, 1, 40, 30, 32, 24))
        np.testing.assert_array_equal(a.mask.labels, b.mask)
