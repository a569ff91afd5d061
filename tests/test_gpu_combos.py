"""Feature combinations on one rotor run: walls on every y / z face,
velocity inflow / outflow in x, Roma or Gaussian spreading, fp64 or fp32
storage, the device path against the C / numpy oracle with the same
extensions switched on (exact arithmetic, host kinematics, 6 steps).
Walls and Gaussian spreading have no reference golden (parity unpinned,
DESIGN.md 8); the Roma / fp64 / no-wall corner of this grid is pinned by
the golden rotor tests.  -m gpu."""

import numpy as np
import pytest

from paper_2402_13171_b200 import Simulation, parse_config
from paper_2402_13171_b200.sim import HostKinematics
from tests.scenarios import oracle_for, rotor_raw, write_rotor_files

pytestmark = pytest.mark.gpu

F32_ULP = 2.0 ** -23
WALLS = {"y_lo": "no_slip", "y_hi": "free_slip", "z_lo": "free_slip", "z_hi": "no_slip"}


def _cfg(tmp_path, precision, spreading):
    write_rotor_files(str(tmp_path), 6)
    raw = rotor_raw((20, 16, 16), (False, False, False), "velocity_inflow_outflow",
                    position=(1.1, 0.9, 0.2), precision=precision)
    raw["run"]["walls"] = dict(WALLS)
    if spreading is not None:
        raw["run"]["spreading"] = {"kernel": "gaussian", "epsilon": spreading}
    return parse_config(raw, base_dir=str(tmp_path))


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("spreading", [None, 1.2])
def test_walled_rotor_vs_oracle(gpu, tmp_path, precision, spreading):
    sim = Simulation(_cfg(tmp_path, precision, spreading), kinematics="host")
    host = HostKinematics(_cfg(tmp_path, precision, spreading))
    ref = oracle_for(host)
    for _ in range(6):
        sim.step()
        ref.step(host.refresh())
        host.advance()
        rho, u, blade = sim._alm_results()
        np.testing.assert_allclose(rho, ref.samples[:, 0], rtol=1e-12)
        np.testing.assert_allclose(u, ref.samples[:, 1:], rtol=1e-10, atol=1e-15)
        np.testing.assert_allclose(blade, ref.blade, rtol=1e-9, atol=1e-12)
    f = np.asarray(sim.fields[0].interior, np.float64)
    F = np.asarray(sim.fields[0].interior_force, np.float64)
    sim.close()
    want_f = np.asarray(ref.interior, np.float64)
    want_F = np.asarray(ref.force[1:-1, 1:-1, 1:-1], np.float64)
    if precision == "double":
        np.testing.assert_allclose(f, want_f, rtol=0, atol=1e-14)
        np.testing.assert_allclose(F, want_F, rtol=1e-12, atol=1e-18)
    else:
        # float32 storage: the trilinear sum order (einsum in the reference,
        # fixed here) moves a force by an ulp at most, and the populations
        # that collide with it by as much
        for got, want in ((f, want_f), (F, want_F)):
            tol = 2 * F32_ULP * np.maximum(np.abs(want), 1e-30)
            assert not (np.abs(got - want) > tol).any(), float(np.abs(got - want).max())
    assert np.isfinite(f).all() and np.abs(F).max() > 0.0   # the rotor forced the flow
