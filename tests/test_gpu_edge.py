"""Actuator edge cases through the device path (the reference's
test_actuator.py contracts at driver level): linear-field sampling,
degenerate flow, zero thrust coefficient, disk thrust formula, points
leaving a non-periodic domain.  -m gpu."""

import numpy as np
import pytest

from paper_2402_13171_b200 import ConfigError, Simulation, parse_config

pytestmark = pytest.mark.gpu

STATIC_BLADE = """
name: b
components:
  - name: root
    position: [2.0, 2.0, 1.5]
  - name: blade
    parent: root
    discretization: {type: line, points: 5, r_end: 0.8, chord: 0.1, polar: flat}
"""
FLAT = "alpha_deg,cl,cd\n-10,1.0,0.2\n10,1.0,0.2\n"


def _cfg(tmp_path, yaml_text, wind=(8.0, 0.0, 0.0), periodic=(True, True, True), extra=None):
    (tmp_path / "t.yaml").write_text(yaml_text)
    (tmp_path / "flat.csv").write_text(FLAT)
    raw = {"domain": {"cells": [16, 16, 16], "periodicity": list(periodic)},
           "fluid": {"kinematic_viscosity": 5.0, "wind": list(wind),
                     "reference_velocity": 8.0},
           "resolution": {"cells_per_diameter": 8, "reference_diameter": 2.0, "mach": 0.1},
           "run": {"steps": 1}, "turbines": [{"file": "t.yaml"}],
           "polars": [{"id": "flat", "file": "flat.csv"}]}
    if extra:
        raw.update(extra)
    return parse_config(raw, base_dir=str(tmp_path))


def test_sampling_reproduces_a_linear_field(gpu, tmp_path):
    """test_actuator.py:163-174: trilinear sampling is exact for a field
    linear in the coordinates (first step samples the initial macro)."""
    cfg = _cfg(tmp_path, STATIC_BLADE)
    sim = Simulation(cfg)
    X, Y, Z = np.meshgrid(*(np.arange(16) + 0.5,) * 3, indexing="ij")
    macro = np.zeros((16, 16, 16, 4))
    macro[..., 0] = 1.0 + 1e-3 * X
    macro[..., 1] = 0.01 + 1e-4 * (2.0 * X - Y + 0.5 * Z)
    macro[..., 2] = -1e-4 * Z
    sim.fields[0].interior_macro = macro
    sim.step()
    rho, u, _ = sim._alm_results()
    pos = sim._kin_view()[:, 0:3]
    np.testing.assert_allclose(rho, 1.0 + 1e-3 * pos[:, 0], rtol=1e-13)
    np.testing.assert_allclose(u[:, 0], 0.01 + 1e-4 * (2.0 * pos[:, 0] - pos[:, 1] +
                                                        0.5 * pos[:, 2]), rtol=1e-12)
    np.testing.assert_allclose(u[:, 1], -1e-4 * pos[:, 2], rtol=1e-12)
    sim.close()


def test_degenerate_flow_gives_zero_force(gpu, tmp_path):
    """test_actuator.py:239-245 / sim.py:227-230: no relative wind, no force."""
    sim = Simulation(_cfg(tmp_path, STATIC_BLADE, wind=(0.0, 0.0, 0.0)))
    sim.step()
    _, _, blade = sim._alm_results()
    assert np.all(blade == 0.0)
    assert np.all(sim.fields[0].interior_force == 0.0)
    sim.close()


DISK = """
name: d
components:
  - name: hub
    position: [2.0, 2.0, 2.0]
    discretization: {type: disk, radius: 1.0, rings: 3, sectors: 8,
                     thrust_coefficient: [0.6, 0.0, 0.4]}
"""


def test_disk_ring_thrust_formula_and_zero_ct(gpu, tmp_path):
    """test_actuator.py:264-305: a ring with C_T = 0 carries no force; each
    ring's total thrust is 1/2 rho u_inf^2 C_T A_ring against the wind."""
    cfg = _cfg(tmp_path, DISK)
    sim = Simulation(cfg)
    sim.step()
    rho, u, blade = sim._alm_results()
    areas = np.array([p.area for p in sim.points])
    u_ax = u[:, 0] * cfg.units.velocity_scale
    rho_p = rho * cfg.units.rho_ref
    for j, ct in enumerate((0.6, 0.0, 0.4)):
        sl = slice(8 * j, 8 * (j + 1))
        A = areas[sl].sum()
        if ct == 0.0:
            assert np.all(blade[sl] == 0.0)
            continue
        a = (1.0 - np.sqrt(1.0 - ct)) / 2.0
        u_d = (u_ax[sl] * areas[sl]).sum() / A
        u_inf = u_d / (1.0 - a)
        thrust = 0.5 * ((rho_p[sl] * areas[sl]).sum() / A) * u_inf ** 2 * ct * A
        # force on the fluid opposes the wind; the blade (disk) force is along it
        np.testing.assert_allclose(blade[sl, 0].sum(), thrust, rtol=1e-12)
        np.testing.assert_allclose(blade[sl, 1:], 0.0, atol=1e-12 * thrust)
    sim.close()


def test_point_leaving_a_non_periodic_domain_raises(gpu, tmp_path):
    """blocks.py:57-70: a point outside a non-periodic axis is a
    ConfigError (device kinematics report it at the next synchronisation)."""
    tip = STATIC_BLADE.replace("position: [2.0, 2.0, 1.5]", "position: [2.0, 2.0, 3.5]")
    tip = tip.replace("r_end: 0.8", "r_end: 0.7")
    cfg = _cfg(tmp_path, tip, periodic=(True, True, False))
    with pytest.raises(ConfigError):
        sim = Simulation(cfg)
        sim.step()
        sim.synchronize()
