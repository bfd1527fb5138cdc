"""Pin the CPU oracle against golden vectors produced by the reference itself.

The fixtures come from `tests/golden/make_golden.py`, which runs the reference
package (`/root/reference/pkg/src/prost`).  The oracle restates the same numpy
operation sequence, so most comparisons are exact.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import prost_oracle as orc


def load(name):
    return np.load(GOLDEN / f"{name}.npz")


def test_cost_and_gradient_bit_exact():
    z = load("cost_vectors")
    for p in (0.25, 0.5, 0.7, 1.0, 2.0):
        key = f"p{p}"
        c, g = orc.lp_cost_grad(z[key + "_r"], p, 1e-4, z[key + "_w"])
        assert c == float(z[key + "_cost"])
        np.testing.assert_array_equal(g, z[key + "_grad"])


def test_fit_bit_exact():
    z = load("fit_vectors")
    for case in range(4):
        key = f"c{case}_"
        p, mu, iters = z[key + "prm"]
        k = z[key + "U"].shape[1]
        prm = orc.OracleParams(k=k, p=p, mu=mu, delta=0.35, max_iters=int(iters))
        y0 = z[key + "y0"]
        y0 = None if np.isnan(y0).all() else y0
        ft = orc.fit(z[key + "U"], z[key + "x"], y0, prm, z[key + "w"])
        np.testing.assert_array_equal(ft.y, z[key + "y"])
        np.testing.assert_array_equal(ft.residual, z[key + "residual"])
        assert ft.cost == float(z[key + "cost"])
        assert [ft.iterations, ft.cost_evals, ft.grad_evals] == list(z[key + "counts"])


def _traj_params(z):
    k, p, mu, delta, omega, t_init, t_min, tau, iters, seed = z["prm"]
    return orc.OracleParams(k=int(k), p=p, mu=mu, delta=delta, omega=omega, t_init=t_init,
                            t_min=t_min, tau=tau, max_iters=int(iters)), int(seed)


def test_step_trajectory_bit_exact():
    z = load("step_trajectory")
    prm, seed = _traj_params(z)
    st = orc.core_init(z["frames"].shape[1], prm, seed)
    np.testing.assert_array_equal(st.U, z["U0"])
    for i, x in enumerate(z["frames"]):
        st, r, ft = orc.core_step(st, x, prm)
        np.testing.assert_array_equal(st.U, z["U"][i])
        np.testing.assert_array_equal(st.y, z["y"][i])
        np.testing.assert_array_equal(st.w, z["w"][i])
        np.testing.assert_array_equal(r, z["residual"][i])
        assert ft.cost == z["cost"][i]
        assert [ft.iterations, ft.cost_evals, ft.grad_evals] == list(z["counts"][i])


def test_periodic_reorthonormalization():
    z = load("qr_chain")
    prm = orc.OracleParams(k=3, p=0.5, mu=0.06125, delta=0.35, omega=5e-5, t_init=1e-2,
                           t_min=1e-3, tau=1e-3, max_iters=2)
    st = orc.core_init(48, prm, 3)
    for i, x in enumerate(z["frames"]):
        st, _, _ = orc.core_step(st, x, prm)
        if f"U{i}" in z:
            np.testing.assert_array_equal(st.U, z[f"U{i}"])
            assert st.since_qr == int(z[f"since{i}"])
    # the reset happens exactly once, at the 1000th geodesic step
    assert int(z["since999"]) == 0 or int(z["since1000"]) == 0


@pytest.mark.parametrize("name", ["push_gray", "push_rgb"])
def test_stream_pipeline_bit_exact(name):
    z = load(name)
    k, p, mu, iters, i_init, seed, channels = z["cfg"]
    prm = orc.OracleParams(k=int(k), p=p, mu=mu, delta=0.35, omega=5e-5, t_init=5e-3,
                           t_min=1e-4, tau=orc.decay_rate(5e-3, 1e-4, int(i_init)),
                           max_iters=int(iters))
    pipe = orc.PipelineOracle(32, 24, int(channels), prm, i_init=int(i_init), seed=int(seed))
    for i, v in enumerate(z["frames"]):
        rec = pipe.push(v)
        np.testing.assert_array_equal(rec.mask, z["mask"][i])
        np.testing.assert_array_equal(rec.raw_mask, z["raw_mask"][i])
        np.testing.assert_array_equal(rec.residual, z["residual"][i])
        assert rec.fit_cost == z["fit_cost"][i]
        assert rec.step == z["step"][i]
        np.testing.assert_array_equal(pipe.background(), z["background"][i])
    np.testing.assert_array_equal(pipe.state.U, z["U"])
    np.testing.assert_array_equal(pipe.norm.mean, z["mean"])
    assert pipe.norm.std == float(z["std"])
