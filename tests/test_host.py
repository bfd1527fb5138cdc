"""CPU tests: the C-ABI library loads and exports the declared symbols, and the
host-side logic (parameter mirrors, validation, generator) behaves like the
reference's.  No device compute here."""

from __future__ import annotations

import ctypes
import math
import re

import numpy as np
import pytest

from conftest import ROOT


def header_functions():
    text = (ROOT / "include" / "prost_b200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|void)\s+(prost_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1302_2073_b200 import _native

    lib = _native.lib()
    declared = header_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.EXPORTS)
    assert lib.prost_abi_version() == 2


def test_struct_layouts_match_header():
    from paper_1302_2073_b200 import _native

    assert ctypes.sizeof(_native.Params) == 8 * 4 + 11 * 8
    assert ctypes.sizeof(_native.FitInfo) == 8 * 3 + 4 * 4
    assert ctypes.sizeof(_native.Outputs) == 5 * 8 + 2 * 4 + 8 + 8  # + fit_residual, fit_async (ABI 2)


def test_create_validates_before_touching_the_device():
    """Invalid parameters are rejected by prost_create with the reference's
    error classes, without needing a GPU."""
    import paper_1302_2073_b200 as pkg
    from paper_1302_2073_b200 import _native
    from paper_1302_2073_b200.params import to_native

    lib = _native.lib()
    good = pkg.ProstParams(k=4, cfg=pkg.LpConfig(p=0.5, mu=1e-4), delta=0.35)
    cases = [
        (dict(k=40), _native.ERR_CONFIG),          # k above the supported maximum
        (dict(channels=2), _native.ERR_DIMENSION),  # channels must be 1 or 3
        (dict(max_backtracks=100), _native.ERR_CONFIG),
        (dict(width=2, height=1, channels=1), _native.ERR_DIMENSION),  # k >= n
        (dict(width=0), _native.ERR_DIMENSION),     # empty frame
        (dict(cg_max_iters=0), _native.ERR_CONFIG),
        (dict(shrink=1.0), _native.ERR_CONFIG),
    ]
    for override, code in cases:
        p = to_native(good, 8, 6, 1, 10)
        for key, val in override.items():
            setattr(p, key, val)
        h = ctypes.c_void_p()
        rc = lib.prost_create(ctypes.byref(p), 1, 0, 0, ctypes.byref(h))
        assert rc == code, (override, rc)
        assert _native.last_error(h)
        lib.prost_destroy(h)
    # an empty batch
    h = ctypes.c_void_p()
    assert lib.prost_create(ctypes.byref(to_native(good, 8, 6, 1, 10)), 0, 0, 0, ctypes.byref(h)) == \
        _native.ERR_CONFIG
    lib.prost_destroy(h)


def test_param_mirrors_match_reference_semantics():
    import paper_1302_2073_b200 as pkg

    with pytest.raises(pkg.ConfigError):
        pkg.LpConfig(p=0.0, mu=1e-3)
    with pytest.raises(pkg.ConfigError):
        pkg.LpConfig(p=0.5, mu=0.0)
    with pytest.raises(pkg.ConfigError):
        pkg.CgOptions(shrink=1.0)
    with pytest.raises(pkg.ConfigError):
        pkg.ProstParams(k=3, cfg=pkg.LpConfig(p=0.5, mu=1e-3), delta=0.35, omega=0.0)
    # tracker.py:90-103 closed forms (reference test_tracker.py:41-53)
    tau = pkg.tau_from_init(5e-3, 1e-4, 1000)
    assert tau == pytest.approx(math.log(50) / 1000, rel=1e-14)
    params = pkg.ProstParams(k=3, cfg=pkg.LpConfig(p=0.5, mu=0.06), delta=0.35, tau=tau)
    assert pkg.step_size(1000, params) == pytest.approx(1e-4, abs=1e-12)
    assert pkg.tau_from_init(1e-3, 1e-3, 50) == 0.0
    # jobs.py:100-105: mu=None couples to delta for p < 1, else 1e-3
    assert pkg.RunConfig(p=0.25).resolved_mu() == pytest.approx(0.35 ** 2 * 0.75)
    assert pkg.RunConfig(p=1.0).resolved_mu() == 1e-3
    assert pkg.smoothing_from_threshold(0.35, 0.5) == pytest.approx(0.06125)


def test_bootstrap_basis_matches_oracle_bit_exact():
    import paper_1302_2073_b200 as pkg
    from oracle import prost_oracle as orc

    z = np.load(ROOT / "tests" / "golden" / "step_trajectory.npz")
    U = pkg.random_orthonormal(z["frames"].shape[1], 4, 7).data
    np.testing.assert_array_equal(U, z["U0"])
    np.testing.assert_array_equal(U, orc.orthonormal_init(z["frames"].shape[1], 4, 7))


def test_frame_containers_validate():
    import paper_1302_2073_b200 as pkg

    with pytest.raises(pkg.DimensionError):
        pkg.FrameBuffer(4, 3, 2, np.zeros(24))
    with pytest.raises(pkg.DimensionError):
        pkg.FrameBuffer(4, 3, 1, np.zeros(11))
    fb = pkg.FrameBuffer(2, 1, 3, np.array([0.0, 0.3, 0.3, 0.6, 0.6, 0.9]))
    np.testing.assert_allclose(fb.to_gray().data, [0.3, 0.6])


def test_synthetic_generator_is_seeded_and_bounded():
    from paper_1302_2073_b200.synth import SceneStream, config_spec

    a = SceneStream(config_spec("C0", 3)).next_frames(4)
    b = SceneStream(config_spec("C0", 3)).next_frames(4)
    c = SceneStream(config_spec("C0", 4)).next_frames(4)
    np.testing.assert_array_equal(a, b)
    assert not np.array_equal(a, c)
    assert a.shape == (4, 160 * 120)
    assert a.min() >= 0.0 and a.max() <= 1.0
    rgb = SceneStream(config_spec("C1", 0)).next_frames(2)
    assert rgb.shape == (2, 320 * 240 * 3)


def test_bench_byte_model():
    import bench

    # C0 2,592,000 B; C1 30,643,200 B; C3 10,368,000 B per stream-frame
    assert bench.b_alg(19200, 15, 19200) == 2_592_000
    assert bench.b_alg(230400, 15, 76800) == 30_643_200
    assert bench.b_alg(76800, 15, 76800) == 10_368_000


def test_u8_unit_formula_is_exact():
    """The kernels' 8-bit conversion (u8_unit, prost_kernels.cuh): q = b * fl(1/255),
    then one FMA-residual correction — equal to the reference's float(b / 255)
    (frameio.py:136: the double product rounded to fp32) for all 256 values.
    FMAs evaluated exactly in rationals, rounded once to fp32."""
    from fractions import Fraction

    def round32(v: Fraction) -> np.float32:
        x = np.float32(float(v))
        cands = [np.nextafter(x, np.float32(-np.inf)), x, np.nextafter(x, np.float32(np.inf))]
        return min(cands, key=lambda c: (abs(Fraction(float(c)) - v),
                                         int(np.array(c, dtype=np.float32).view(np.uint32)) & 1))

    def fma(a, b, c):
        return round32(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))

    r = np.float32(1.0 / 255.0)
    for b in range(256):
        bf = np.float32(b)
        q = np.float32(bf * r)
        got = fma(fma(-q, np.float32(255.0), bf), r, q)
        assert got == np.float32(b * (1.0 / 255.0)), b
